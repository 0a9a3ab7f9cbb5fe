"""Pins for the oracle's trace normalisation (O-1..O-6): stable arrival sort
(S:46), touch order, prev / delta against a brute-force scan, SPEC interarrival
examples, group ranking and the chain check."""
import numpy as np
import pytest

import kareto_inputs as ki
from oracle import oracle as O
from tests import brute
from tests.conftest import assign_groups, chains_from_labels


def _random_labels(rng, n_req):
    chains = []
    for _ in range(n_req):
        depth = int(rng.integers(1, 7))
        ch = [int(rng.integers(0, 3))]
        for d in range(depth - 1):
            ch.append(int(rng.integers(0, 3)) + 100 * (d + 1))
        chains.append(ch)
    inc = np.array([0, 0, 1, 2, 3, 5, 8])
    arr = np.cumsum(inc[rng.integers(0, len(inc), n_req)])
    perm = rng.permutation(n_req)
    return [chains[i] for i in perm], arr[perm]


def test_prev_delta_match_brute_force(rng):
    for _ in range(40):
        chains, arr = _random_labels(rng, int(rng.integers(5, 40)))
        tr = ki.from_chains(chains, arr)
        ot = O.OracleTrace(tr, top_k=2)
        e = ot.export()
        sc = chains_from_labels(chains, arr)
        prev, delta = brute.prev_delta(sc)
        assert np.array_equal(e["prev"], prev)
        assert np.array_equal(e["delta"], delta)
        # sum over groups of #Delta_g = N - U
        assert ot.reuse_g.sum() == ot.N - ot.U
        assert ot.U_g.sum() == ot.U


def test_stable_sort_by_arrival_then_file_index():
    # three requests, equal arrivals keep file order; single distinct blocks each
    tr = ki.from_chains([[5], [6], [7]], [10, 0, 10])
    e = O.OracleTrace(tr).export()
    # sorted order: file 1 (t=0), file 0 (t=10), file 2 (t=10)
    h5, h6, h7 = (O.chain_hashes(ki._block_tokens(x))[0] for x in (5, 6, 7))
    assert list(e["hash"]) == [h6, h5, h7]


def test_touch_order_is_leaf_to_root():
    tr = ki.from_chains([[1, 2, 3]], [0])
    e = O.OracleTrace(tr).export()
    assert list(e["k"]) == [2, 1, 0]


def test_spec_interarrival_examples():
    # S:79  block accessed at t = {0, 5, 5} -> intervals {5, 0}
    tr = ki.from_chains([[9], [9], [9]], [0, 5, 5])
    e = O.OracleTrace(tr).export()
    assert sorted(int(x) for x in e["delta"] if x >= 0) == [0, 5]
    # S:185 one block accessed at {0, 4, 10} -> {4, 6}
    tr = ki.from_chains([[9], [9], [9]], [0, 4, 10])
    e = O.OracleTrace(tr).export()
    assert [int(x) for x in e["delta"] if x >= 0] == [4, 6]


def test_group_ranking_spec_examples():
    # S:175 two subtrees with reuse 10 and 3, K = 1 -> group 0 is the 10-reuse subtree
    chains = [[1, 11]] * 6 + [[2, 12]] * 3  # root 1: 5 reuses x2 blocks = 10; root 2: 2 x 2 = 4
    chains = [[1, 11]] * 6 + [[2]] * 4      # root 1: 10 reuses; root 2: 3 reuses
    arr = list(range(len(chains)))
    ot = O.OracleTrace(ki.from_chains(chains, arr), top_k=1)
    e = ot.export()
    # requests 0..5 root 1 -> group 0 ; requests 6..9 root 2 -> residual group 1
    assert list(e["group"]) == [0] * 6 + [1] * 4
    assert list(ot.reuse_g) == [10, 3]
    # S:174 one subtree, K = 3 -> 1 real group + empty residual (residual always exists)
    ot = O.OracleTrace(ki.from_chains([[1, 2], [1, 3]], [0, 1]), top_k=3)
    assert list(ot.U_g) == [3, 0, 0, 0] and list(ot.reuse_g) == [1, 0, 0, 0]


def test_groups_match_independent_tally(rng):
    for _ in range(30):
        chains, arr = _random_labels(rng, int(rng.integers(5, 40)))
        tr = ki.from_chains(chains, arr)
        K = int(rng.integers(0, 4))
        ot = O.OracleTrace(tr, top_k=K)
        e = ot.export()
        sc = chains_from_labels(chains, arr)
        root_hash = {}
        for (_a, _g, ch) in sc:
            root_hash[ch[0]] = int(O.chain_hashes(ki._block_tokens(ch[0][0]))[0])
        sg = assign_groups(sc, K, root_hash)
        assert list(e["group"]) == [g for (_a, g, _c) in sg]


def test_chain_violation_rejected_in_hash_mode():
    # block 0xB appears once as a root and once as a child: not chain-consistent (S7 / O-4)
    tr = ki.Trace(np.array([0, 1], np.int64), np.array([1, 1], np.int32), np.array([0, 1, 3], np.int64),
                  block_hash=np.array([0xB, 0xA, 0xB], np.uint64))
    with pytest.raises(O.OracleError) as ei:
        O.OracleTrace(tr, mode="hashes")
    assert ei.value.status == O.E_CHAIN
    # two different parents for the same child hash
    tr = ki.Trace(np.array([0, 1], np.int64), np.array([1, 1], np.int32), np.array([0, 2, 4], np.int64),
                  block_hash=np.array([0xA, 0xC, 0xB, 0xC], np.uint64))
    with pytest.raises(O.OracleError):
        O.OracleTrace(tr, mode="hashes")


def test_hash_mode_equals_token_mode_given_the_same_hashes(rng):
    chains, arr = _random_labels(rng, 30)
    tr = ki.from_chains(chains, arr)
    bh, boff = [], [0]
    for r in range(tr.n_requests):
        h = O.chain_hashes(tr.tokens[tr.offsets[r]:tr.offsets[r + 1]])
        bh.append(h)
        boff.append(boff[-1] + len(h))
    th = ki.Trace(tr.arrival_ms, tr.output_tokens, np.array(boff, np.int64), block_hash=np.concatenate(bh),
                  input_tokens=np.diff(tr.offsets))
    a = O.OracleTrace(tr).export()
    b = O.OracleTrace(th, mode="hashes").export()
    for k in ("hash", "prev", "delta", "req", "k", "group"):
        assert np.array_equal(a[k], b[k]), k


def test_invalid_inputs():
    with pytest.raises(O.OracleError):
        O.OracleTrace(ki.Trace(np.zeros(0, np.int64), np.zeros(0, np.int32), np.zeros(1, np.int64),
                               tokens=np.zeros(0, np.uint32)))
    with pytest.raises(O.OracleError):
        O.OracleTrace(ki.Trace(np.zeros(1, np.int64), np.array([-1], np.int32), np.array([0, 16], np.int64),
                               tokens=np.zeros(16, np.uint32)))

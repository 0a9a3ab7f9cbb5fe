"""Pins for O1, the oracle's literal per-configuration replay (R9-R24):
worked example W1, Belady's textbook strings (Belady 1969; Mattson et al. 1970),
SPEC tiered_store examples, the LRU stack/inclusion property,
the paper's closed forms H_g / C_g, and a naive
brute-force replay (tests/brute.py) on random chain-consistent traces."""
import numpy as np
import pytest

import kareto_inputs as ki
from oracle import oracle as O
from tests import brute
from tests.conftest import assign_groups, chains_from_labels

INF = O.INF_CAP
POL = {"lru": O.LRU, "fifo": O.FIFO, "lfu": O.LFU}


def run(chains, arr, caps, policy="lru", ttl=None, K=0):
    ot = O.OracleTrace(ki.from_chains(chains, arr), top_k=K)
    cf = O.configs(caps, policy=POL[policy])
    if ttl is not None:
        ttl = np.asarray(ttl, np.uint32).reshape(1, -1)
    return ot.replay(cf, ttl)


def as_dict(c):
    return dict(hit=[int(x) for x in c["hit"]], miss=int(c["miss"]), evict=[int(x) for x in c["evict"]],
                disk_writes=int(c["disk_writes"]), hit_pos_sum=int(c["hit_pos_sum"]),
                bytetime_block_ms=int(c["bytetime_block_ms"]), resident_after_hole=int(c["resident_after_hole"]))


W1 = ([[1, 2, 3], [1, 2, 4], [1, 2, 3]], [0, 10, 20])


def test_w1_worked_example():
    # SURVEY 8.c.8 W1 (verified there by brute force)
    c = as_dict(run(*W1, [[1, 1, 1]])[0])
    assert c["hit"] == [2, 2, 0] and c["miss"] == 5 and c["evict"] == [8, 7, 2]
    c = as_dict(run(*W1, [[1, 1, 2]])[0])
    assert c["hit"] == [2, 2, 1] and c["miss"] == 4 and c["evict"] == [8, 7, 0]
    c = as_dict(run(*W1, [[1, 1, 2]], ttl=[15])[0])
    assert c["hit"] == [2, 2, 0] and c["miss"] == 5  # disk hit lost: delta_C = 20 > 15
    c = as_dict(run(*W1, [[0, 0, INF]], ttl=[15])[0])
    # TTL mode: h3 = H(15) with Delta = {10,10,10,10,20}, U = 4; bytetime = C(15) = 4*15 + 55
    assert c["hit"][2] == 4 and c["bytetime_block_ms"] == 115


BELADY = [1, 2, 3, 4, 1, 2, 5, 1, 2, 3, 4, 5]


@pytest.mark.parametrize("policy,c1,hits", [("lru", 3, 2), ("lru", 4, 4), ("fifo", 3, 3), ("fifo", 4, 2),
                                            ("lfu", 3, 2), ("lfu", 4, 4)])
def test_belady_string_single_tier(policy, c1, hits):
    # Belady (1969): FIFO with 3 frames faults 9 times, with 4 frames 10 times (the anomaly);
    # LRU faults 10 / 8 times.  Single tier: c2 = c3 = 0.
    chains = [[x] for x in BELADY]
    c = as_dict(run(chains, list(range(12)), [[c1, 0, 0]], policy)[0])
    assert sum(c["hit"]) == hits
    assert c["miss"] == 12 - hits


@pytest.mark.parametrize("policy,hits", [("lru", 2), ("fifo", 1), ("lfu", 2)])
def test_w3_abaca(policy, hits):
    chains = [[x] for x in [1, 2, 1, 3, 1]]
    c = as_dict(run(chains, list(range(5)), [[2, 0, 0]], policy)[0])
    assert sum(c["hit"]) == hits


def test_spec_lookup_example_s243():
    # "4-block chain with blocks 1-2 in DRAM, 3 on disk, 4 absent -> (hbm 0, dram 2, disk 1)"
    # Build that state: touch [a,b,c] (c1=0: everything cascades), then a filler chain pushes
    # them down; c2 = 2 keeps a, b in DRAM (root-first order) and c lands on disk.
    chains = [[1, 2, 3], [1, 2, 3, 4]]
    c = as_dict(run(chains, [0, 1], [[0, 2, 5]])[0])
    assert c["hit"][:3] == [0, 2, 1]


def test_spec_lru_victim_s253():
    # "capacity 2 blocks, admit a,b,c sequentially -> evicts a (LRU)": afterwards b, c hit, a misses
    chains = [[1], [2], [3], [2], [3], [1]]
    c = as_dict(run(chains, list(range(6)), [[2, 0, 0]])[0])
    assert sum(c["hit"]) == 2 and c["evict"][0] == 2  # a (t=0), then b at the final admit


def _random(rng, n_req=None):
    n = n_req or int(rng.integers(5, 41))
    chains = []
    for _ in range(n):
        depth = int(rng.integers(1, 7))
        ch = [int(rng.integers(0, 3))]
        for d in range(depth - 1):
            ch.append(int(rng.integers(0, 3)) + 100 * (d + 1))
        chains.append(ch)
    inc = np.array([0, 0, 1, 2, 3, 5, 8])
    arr = np.cumsum(inc[rng.integers(0, len(inc), n)])
    perm = rng.permutation(n)
    return [chains[i] for i in perm], arr[perm]


def _brute_input(chains, arr, K):
    sc = chains_from_labels(chains, arr)
    rh = {ch[0]: int(O.chain_hashes(ki._block_tokens(ch[0][0]))[0]) for (_a, _g, ch) in sc}
    return assign_groups(sc, K, rh)


def test_replay_matches_brute_force_all_policies_and_modes(rng):
    taus = [None, 0, 1, 3, 6, 50]
    for trial in range(60):
        chains, arr = _random(rng)
        K = int(rng.integers(0, 3))
        ot = O.OracleTrace(ki.from_chains(chains, arr), top_k=K)
        sg = _brute_input(chains, arr, K)
        for _ in range(6):
            policy = ["lru", "fifo", "lfu"][int(rng.integers(0, 3))]
            ttl_mode = rng.random() < 0.3
            c1, c2, c3 = (int(x) for x in rng.integers(0, 6, 3))
            if ttl_mode:
                tau = [int(rng.choice([0, 1, 3, 6, 50])) for _ in range(K + 1)]
                caps = (c1, c2, None)
            else:
                tau = [taus[int(rng.integers(0, len(taus)))] for _ in range(K + 1)]
                caps = (c1, c2, c3)
            want = brute.replay(sg, caps, policy, tau)
            cf = O.configs([[c1, c2, INF if ttl_mode else c3]], policy=POL[policy])
            row = np.array([[0xFFFFFFFF if t is None else t for t in tau]], np.uint32)
            got = as_dict(ot.replay(cf, row)[0])
            assert got == want, (trial, policy, caps, tau)


def test_lru_inclusion_property(rng):
    # LRU is a stack algorithm on a fixed reference string (Mattson et al. 1970):
    # h1 nondecreasing in c1, h1+h2 in c1+c2, total hits in c1+c2+c3.
    for _ in range(20):
        chains, arr = _random(rng)
        ot = O.OracleTrace(ki.from_chains(chains, arr))
        caps = [[a, b, c] for a in range(5) for b in range(4) for c in range(4)]
        cnt = ot.replay(O.configs(caps))
        by = {tuple(k): c for k, c in zip(caps, cnt)}
        for (a, b, c), x in by.items():
            if (a + 1, b, c) in by:
                assert by[(a + 1, b, c)]["hit"][0] >= x["hit"][0]
            if (a, b + 1, c) in by:
                y = by[(a, b + 1, c)]
                assert y["hit"][0] + y["hit"][1] >= x["hit"][0] + x["hit"][1]
            if (a, b, c + 1) in by:
                assert by[(a, b, c + 1)]["hit"].sum() >= x["hit"].sum()
            # totals depend only on c1+c2+c3 (single LRU stack)
        tot = {}
        for (a, b, c), x in by.items():
            tot.setdefault(a + b + c, set()).add(int(x["hit"].sum()))
        assert all(len(v) == 1 for v in tot.values())


def test_conservation_and_prefix_closure(rng):
    for _ in range(20):
        chains, arr = _random(rng)
        ot = O.OracleTrace(ki.from_chains(chains, arr))
        for pol in (O.LRU, O.FIFO, O.LFU):
            cf = O.configs([[1, 2, 3], [0, 1, 0], [2, 0, 4]], policy=pol)
            for c in ot.replay(cf):
                assert int(c["hit"].sum()) + int(c["miss"]) == ot.N
                if pol != O.FIFO:
                    assert int(c["resident_after_hole"]) == 0  # LRU / LFU residency is prefix-closed


def test_ttl_mode_closed_forms_H_and_C(rng):
    # c1 = c2 = 0 in TTL mode: disk hits == sum_g H_g(tau_g) and bytetime == sum_g C_g(tau_g)
    # with H_g(t) = #{delta <= t}, C_g(t) = |B_g| t + sum min(t, delta)
    for _ in range(30):
        chains, arr = _random(rng)
        K = int(rng.integers(0, 3))
        ot = O.OracleTrace(ki.from_chains(chains, arr), top_k=K)
        e = ot.export()
        tau = rng.choice([0, 1, 3, 6, 50], K + 1).astype(np.uint32)
        cf = O.configs([[0, 0, INF]])
        c = ot.replay(cf, tau.reshape(1, -1))[0]
        H = C = 0
        for g in range(K + 1):
            sel = (e["prev"] >= 0) & (e["group"][e["req"]] == g)
            d = e["delta"][sel]
            H += int((d <= tau[g]).sum())
            C += int(ot.U_g[g]) * int(tau[g]) + int(np.minimum(d, tau[g]).sum())
        assert int(c["hit"][2]) == H
        assert int(c["bytetime_block_ms"]) == C


def test_spec_group_curve_numbers():
    # Delta = {1,3,3,7}: H(0)=0, H(3)=3, H(inf)=4; |B|=2: C(3) = 2*3 + (1+3+3+3) = 16.
    # One block 'x' reused at +1, +3, +3, +7 ms plus an unrelated single-use block 'y' -> |B| = 2.
    chains = [[1], [1], [1], [1], [1], [2]]
    arr = [0, 1, 4, 7, 14, 14]
    for tau, H, C in [(0, 0, 0 + 0), (3, 3, 16), (1_000_000, 4, None)]:
        c = run(chains, arr, [[0, 0, INF]], ttl=[tau])[0]
        assert int(c["hit"][2]) == H
        if C is not None:
            assert int(c["bytetime_block_ms"]) == C


def test_invalid_configs():
    ot = O.OracleTrace(ki.from_chains([[1]], [0]))
    with pytest.raises(O.OracleError):
        ot.replay(O.configs([[1, 1, INF]]))  # TTL mode with tau = infinity (R22)
    with pytest.raises(O.OracleError):
        ot.replay(O.configs([[1, 1, 1]], policy=3))

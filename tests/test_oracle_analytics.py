"""Pins for the trace-analytics oracle (oracle/analytics.py, row f4): X6 reuse skew / Lorenz curve
 and X5 oracle-TTL footprint.

Pinned against: SPEC's worked cases, an independent tally of hits with
numpy.unique over the chained hashes, and a brute-force footprint from the set definition
(a block is active after request r iff it has an access at or before r and one after r)."""
import numpy as np
import pytest

import kareto_inputs as ki
from oracle import analytics as X
from oracle import oracle as O


def export(tr, top_k=2):
    ot = O.OracleTrace(tr, top_k=top_k)
    return ot.export(), ot.R


def test_every_block_reused_once_is_the_diagonal():
    # 10 distinct single-block requests, each repeated once later
    chains = [[i] for i in range(10)] + [[i] for i in range(10)]
    e, _ = export(ki.from_chains(chains, list(range(20))))
    T, k90, f90, lor, U = X.skew(e, n_pts=11)
    assert (T, U, k90) == (10, 10, 9) and f90 == 0.9
    assert lor == [i / 10 for i in range(11)]


def test_one_block_holds_all_reuse():
    # 100 distinct blocks, block 0 re-accessed 5 times
    chains = [[i] for i in range(100)] + [[0]] * 5
    e, _ = export(ki.from_chains(chains, list(range(105))))
    T, k90, f90, lor, U = X.skew(e)
    assert (T, U, k90) == (5, 100, 1) and f90 == 0.01
    assert lor[0] == 0.0 and lor[-1] == 1.0 and lor[1] == 1.0


def test_no_reuse():
    e, R = export(ki.from_chains([[i] for i in range(6)], list(range(6))))
    T, k90, f90, lor, U = X.skew(e)
    assert T == 0 and f90 == 1.0 and all(v == 0.0 for v in lor)
    cum, act = X.footprint(e, R)
    assert cum.tolist() == [1, 2, 3, 4, 5, 6] and act.tolist() == [0] * 6


def test_single_block_interval():
    # block accessed at request 0 (t = 0) and request 2 (t = 10); an unrelated block at t = 5
    e, R = export(ki.from_chains([[7], [8], [7]], [0, 5, 10]))
    cum, act = X.footprint(e, R)
    assert cum.tolist() == [1, 2, 2] and act.tolist() == [1, 1, 0]


def brute_footprint(e, R):
    first, last = {}, {}
    for h, r in zip(e["hash"].tolist(), e["req"].tolist()):
        first[h] = min(first.get(h, r), r)
        last[h] = max(last.get(h, r), r)
    acc = {}
    for h, r in zip(e["hash"].tolist(), e["req"].tolist()):
        acc.setdefault(h, set()).add(r)
    cum = [sum(1 for h in first if first[h] <= r) for r in range(R)]
    act = [sum(1 for h in acc if any(x <= r for x in acc[h]) and any(x > r for x in acc[h])) for r in range(R)]
    return cum, act


def test_against_tally_and_brute_force():
    rng = np.random.default_rng(5)
    for trial in range(25):
        tr = ki.random_prefix_tree(rng)
        e, R = export(tr)
        _, counts = np.unique(e["hash"], return_counts=True)
        hits = np.sort(counts - 1)[::-1]
        T, k90, f90, lor, U = X.skew(e)
        assert (T, U) == (int(hits.sum()), len(hits))
        if T:
            c = np.cumsum(hits)
            assert k90 == int(np.argmax(10 * c >= 9 * T)) + 1
            assert lor[0] == 0.0 and lor[-1] == 1.0 and all(a <= b for a, b in zip(lor, lor[1:]))
        cum, act = X.footprint(e, R)
        bc, ba = brute_footprint(e, R)
        assert cum.tolist() == bc and act.tolist() == ba


def test_chat_trace_skew_is_sane():
    e, R = export(ki.synthetic("chat", R=300, seed=0))
    T, k90, f90, lor, U = X.skew(e)
    assert 0 < f90 < 1 and T == int((e["prev"] >= 0).sum())

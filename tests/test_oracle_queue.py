"""Pins for the row-f3 oracle (oracle/queue.py): per-request tier hits (R49), the FCFS queue with
disk prefetch during queueing (R50-R52) and the TTFT statistics (R53).

Pinned against: the stack path's totals (O2 closed forms, themselves pinned to the literal replay),
the Lindley recursion for one instance, the fluid model's mean TTFT when nothing queues and no
disk is configured, Obs. 2 / Obs. 4 as exact limiting properties (an idle system realises no
disk hits; a saturated one realises them all), and numpy's inverted-CDF percentile."""
import numpy as np
import pytest

import kareto_inputs as ki
from oracle import oracle as O
from oracle import queue as Q

INF = int(O.INF_CAP)


def setup(tr, top_k=2):
    ot = O.OracleTrace(tr, top_k=top_k)
    e = ot.export()
    d, _ = ot.depth()
    return ot, e, d


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_literal_prefixes_match_the_stack_shape(seed):
    # O1's per-request hit prefixes (any policy) against the O2 depth counts for LRU stack configs:
    # same blocks, HBM first, then DRAM, then disk
    tr = ki.synthetic("chat", R=300, seed=seed)
    ot, e, d = setup(tr)
    U = ot.U
    ttl = np.array([[600_000] * 3, [0xFFFFFFFF] * 3], np.uint32)
    for cap, tuner in [((U // 50, U // 10, U // 3), 1), ((U // 20, U // 5, U // 2), 0), ((U // 20, 0, INF), 0),
                       ((0, U // 7, INF), 0)]:
        cf = O.configs([cap], tuner=tuner)
        _, lt = ot.replay_lookup(cf, ttl)
        lit = Q.prefixes_from_lookup(lt.tolist(), e["s"].tolist())
        h1, h2, h3 = Q.per_request_hits(d, e["delta"], e["s"].tolist(), e["group"].tolist(), cap, ttl[tuner])
        assert lit == Q.prefixes_from_counts(h1, h2, h3)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_per_request_hits_sum_to_stack_totals(seed):
    tr = ki.synthetic("chat", R=400, seed=seed)
    ot, e, d = setup(tr)
    U = ot.U
    caps = [(U // 50, U // 10, U // 3), (0, U // 5, 0), (U // 20, 0, INF), (0, 0, INF)]
    ttl = np.array([[600_000] * 3, [0xFFFFFFFF] * 3], np.uint32)
    for tuner in (0, 1):
        for cap in caps:
            if cap[2] == INF and tuner == 1:
                continue
            cf = O.configs([cap], tuner=tuner)
            want = ot.stack_counts(cf, ttl)[0]
            h1, h2, h3 = Q.per_request_hits(d, e["delta"], e["s"].tolist(), e["group"].tolist(), cap, ttl[tuner])
            assert (sum(h1), sum(h2), sum(h3)) == tuple(int(x) for x in want["hit"])


def run(tr, cap, model, ttl=None):
    ot, _, _ = setup(tr)
    return Q.evaluate(tr, ot, O.configs([cap]), ttl, model)[0]


def test_idle_system_realises_no_disk_hits():
    # Obs. 2: requests one hour apart never queue, so no disk block is prefetched in time
    rng = np.random.default_rng(3)
    chains = [[int(rng.integers(0, 3))] + [int(x) for x in rng.integers(0, 4, size=5)] for _ in range(40)]
    tr = ki.from_chains(chains, [3_600_000 * i for i in range(40)], [50] * 40)
    res = run(tr, (0, 0, 1000), O.Model(instances=1))
    assert res["disk_cap"] > 0 and res["disk_real"] == 0


def test_saturated_system_realises_all_disk_hits_and_lindley():
    # Obs. 4: everything arrives at t = 0 on one instance and each request decodes 5000 tokens
    # (0.75 s), so every request after the first waits long enough to load its disk prefix
    rng = np.random.default_rng(4)
    chains = [[int(rng.integers(0, 2))] + [int(x) for x in rng.integers(0, 3, size=8)] for _ in range(30)]
    tr = ki.from_chains(chains, [0] * 30, [5000] * 30)
    m = O.Model(instances=1)
    ot, e, d = setup(tr)
    res = Q.evaluate(tr, ot, O.configs([(0, 0, 1000)]), None, m)[0]
    arr, L, o = Q.request_arrays(tr)
    h1, h2, h3 = Q.per_request_hits(d, e["delta"], e["s"].tolist(), e["group"].tolist(), (0, 0, 1000),
                                    [0xFFFFFFFF] * 3)
    assert res["disk_cap"] > 0 and res["disk_real"] == res["disk_cap"]
    # Lindley recursion with an independently summed prefill (per-token alpha + beta * position over
    # the recomputed positions 16 H .. L-1): TTFT_r = w_r + prefill_r (+ no DRAM here)
    w = 0.0
    for r in range(len(arr)):
        H = h1[r] + h2[r] + h3[r]
        prefill = sum(m.alpha_ps + m.beta_ps * p for p in range(16 * H, int(L[r]))) * 1e-12
        assert res["ttft"][r] == pytest.approx(w + prefill, rel=1e-9, abs=1e-12)
        service = prefill + m.dec_ps * int(o[r]) * 1e-12
        nxt = arr[r + 1] if r + 1 < len(arr) else arr[r]
        w = max(0.0, w + service - (nxt - arr[r]) * 1e-3)


def test_no_queueing_no_disk_matches_fluid_mean():
    tr = ki.synthetic("chat", R=300, seed=5)
    ot, _, _ = setup(tr)
    U = ot.U
    cap = (U // 40, U // 8, 0)
    cf = O.configs([cap])
    m = O.Model(instances=10_000)                 # never queues
    res = Q.evaluate(tr, ot, cf, None, m)[0]
    fluid = ot.objective(m, cf, ot.stack_counts(cf))[0]
    assert res["disk_real"] == res["disk_cap"] == 0
    assert res["mean_ms"] == pytest.approx(fluid[0], rel=1e-12)
    # the fluid makespan is max(span, busy / I); the queue's also waits for the last request to finish
    span_s = ot.span_ms * 1e-3
    assert span_s <= res["makespan_s"] <= span_s + 60.0
    assert res["tok_per_s"] == (ot.Ltok + ot.O) / res["makespan_s"] <= -fluid[1]


def test_realised_prefix_rule():
    # R51 on hand sequences: disk blocks stream in chain order; the prefix ends at the first one
    # not loaded; x = 1.5 loads one disk block
    assert Q.realised([1, 1, 2, 3, 3], 1.5) == (4, 1, 1, 2)
    assert Q.realised([1, 3, 1, 3, 2], 1.0) == (3, 0, 1, 2)       # mixed tiers (FIFO / LFU)
    assert Q.realised([3, 1, 2], 0.0) == (0, 0, 0, 1)
    assert Q.realised([1, 2, 2], 0.0) == (3, 2, 0, 0)


def test_p99_is_the_nearest_rank():
    tr = ki.synthetic("chat", R=257, seed=6)
    res = run(tr, (100, 1000, INF), O.Model(instances=2), np.array([[60_000] * 3], np.uint32))
    assert res["p99_ms"] == 1e3 * np.percentile(res["ttft"], 99, method="inverted_cdf")
    assert res["mean_ms"] == pytest.approx(1e3 * np.mean(res["ttft"]), rel=1e-12)

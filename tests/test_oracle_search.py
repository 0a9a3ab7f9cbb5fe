"""Pins for the row-f1 oracle (oracle/search.py): Alg. 1 adaptive Pareto exploration
 and the exact 3-D hypervolume.

Pinned against things other than the oracle itself: the SPEC's worked hypervolume examples
(tests/golden/hypervolume.json), a closed-form staircase, brute-force cell counting, a Monte
Carlo estimate, hypervolume monotonicity, and hand-traced runs of Alg. 1 on synthetic
landscapes (flat, one latency cliff, a diminishing-return DRAM curve)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import search as S
from tests import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden", "hypervolume.json")


# ------------------------------------------------------------------ hypervolume
def test_hv_golden_examples():
    for ex in json.load(open(GOLD))["examples"]:
        assert S.hypervolume(ex["points"], ex["ref"]) == pytest.approx(ex["hv"], rel=1e-15), ex["cite"]


def test_hv_staircase_closed_form():
    # 2-D unit staircase (i, n-1-i), ref (n, n): area n(n+1)/2; lifted to 3-D with z = 0, ref_z = 1
    for n in (1, 2, 5, 17):
        pts = [(i, n - 1 - i, 0.0) for i in range(n)]
        assert S.hypervolume(pts, (n, n, 1.0)) == n * (n + 1) / 2


def test_hv_brute_force_cells():
    rng = np.random.default_rng(1)
    for trial in range(60):
        n = int(rng.integers(1, 9))
        pts = rng.integers(0, 6, size=(n, 3)).astype(float) if trial % 2 else rng.random((n, 3))
        ref = (7.0, 7.0, 7.0) if trial % 2 else (1.5, 1.2, 1.1)
        assert S.hypervolume(pts, ref) == pytest.approx(brute.hypervolume_cells(pts.tolist(), ref), rel=1e-12)


def test_hv_monte_carlo():
    # 50 random 3-d points within 1% of a Monte Carlo estimate
    rng = np.random.default_rng(7)
    pts = rng.random((50, 3))
    ref = np.array([1.0, 1.0, 1.0])
    x = rng.random((2_000_000, 3))
    dom = np.zeros(len(x), bool)
    for p in pts:
        dom |= np.all(x >= p, axis=1)
    assert S.hypervolume(pts, ref) == pytest.approx(dom.mean(), rel=0.01)


def test_hv_monotone_and_dominated_point():
    rng = np.random.default_rng(3)
    pts = rng.random((20, 3))
    ref = (1.0, 1.0, 1.0)
    hv = S.hypervolume(pts, ref)
    worse = pts[0] + 0.5 * (1 - pts[0])              # dominated by pts[0]
    assert S.hypervolume(np.vstack([pts, worse]), ref) == pytest.approx(hv, rel=1e-14)
    for q in rng.random((10, 3)):
        assert S.hypervolume(np.vstack([pts, q]), ref) >= hv - 1e-15


def test_hv_reference_must_be_strictly_worse():
    with pytest.raises(ValueError, match="point 1"):
        S.hypervolume([(0, 0, 0), (1, 0.5, 0.5)], (1, 1, 1))


# ------------------------------------------------------------------ Alg. 1
def landscape(f_lat, f_cost=lambda d, t: 1.0, f_thr=lambda d, t: -1.0):
    calls = []

    def ev(C):
        calls.append(list(C))
        return [(f_lat(d, t), f_thr(d, t), f_cost(d, t)) for d, t in C]
    return ev, calls


def test_flat_landscape_evaluates_only_the_coarse_grid():
    ev, calls = landscape(lambda d, t: 5.0)
    p = S.SearchParams(0, 2048, 512, 0, 2400, 600)
    log, F, trunc = S.adaptive_search(ev, p)
    assert len(calls) == 1 and len(log) == 25 and not trunc      # 5 x 5 seed grid
    assert {(d, t) for d, t, _ in log} == {(d, t) for d in range(0, 2049, 512) for t in range(0, 2401, 600)}


def test_latency_cliff_is_bisected():
    # hand trace: 2x2 seed {0,100}^2, latency 10 below d = 50 and 1 above, cost 1 + d.
    # round 1: the seed; round 2: midpoints (50, t) of the cliff pairs and the expansion column
    # d = 200 (latency fell 90% between d = 0 and 100 at t = 0); later rounds bisect (0, 50)
    # down to the 1-GB resolution: 25, 37, 43, 46, 48, 49.
    ev, calls = landscape(lambda d, t: 10.0 if d < 50 else 1.0, f_cost=lambda d, t: 1.0 + d)
    log, F, trunc = S.adaptive_search(ev, S.SearchParams(0, 100, 100, 0, 100, 100))
    assert sorted(calls[1]) == [(50, 0), (50, 100), (200, 0), (200, 100)]
    ds = sorted({d for d, _, _ in log})
    assert ds == [0, 25, 37, 43, 46, 48, 49, 50, 100, 200]
    assert len(log) == 2 * len(ds) and not trunc
    assert [len(c) for c in calls] == [4, 4, 2, 2, 2, 2, 2, 2]


def test_dram_expansion_stops_at_the_diminishing_return_threshold():
    f = lambda d: 1.0 + 1e4 / (100.0 + d)                 # convex, decreasing latency in DRAM
    ev, calls = landscape(lambda d, t: f(d))              # constant cost: no refinement
    p = S.SearchParams(0, 200, 100, 0, 600, 600, tau_e=0.05)
    log, F, trunc = S.adaptive_search(ev, p)
    dmax = max(d for d, _, _ in log)
    gain = lambda d: (f(d - 100) - f(d)) / f(d - 100)
    assert gain(dmax) <= 0.05                              # stopped at the first column below tau_e
    assert all(gain(d) > 0.05 for d in range(200, dmax, 100))
    for d in range(0, dmax + 1, 100):                      # every expansion adds the whole TTL column
        assert {(d, 0), (d, 600)} <= {(x, t) for x, t, _ in log}


def test_budget_truncation_and_fine_grid_bound():
    rng = np.random.default_rng(0)
    w = rng.random(4)
    lat = lambda d, t: 1 + w[0] * np.exp(-d / 700) + w[1] * np.exp(-t / 900) + 0.3 * (d > 1500)
    ev, _ = landscape(lat, f_cost=lambda d, t: 1 + d / 100 + t / 300, f_thr=lambda d, t: -1 / lat(d, t))
    p = S.SearchParams(0, 2048, 512, 0, 2400, 600)
    log, F, trunc = S.adaptive_search(ev, p)
    assert not trunc
    dmax = max(d for d, _, _ in log)
    assert len(log) <= (dmax + 1) * (2400 + 1)            # never more than the 1-GB x 1-s fine grid
    st = O.pareto(F)
    for i in np.flatnonzero(st == 1):                      # frontier points are nondominated in the set
        assert not np.any(np.all(F <= F[i], 1) & np.any(F < F[i], 1))
    p2 = S.SearchParams(0, 2048, 512, 0, 2400, 600, max_evals=len(log) - 1)
    log2, _, trunc2 = S.adaptive_search(ev, p2)
    assert trunc2 and len(log2) < len(log) and log2 == log[:len(log2)]


def test_trace_evaluator_matches_literal_replay():
    import kareto_inputs as ki
    tr = ki.synthetic("chat", R=300, seed=2)
    ot = O.OracleTrace(tr, top_k=4)
    m = O.Model()
    ev = S.trace_evaluator(ot, m, hbm_gb=0.05, block_bytes=m.block_bytes)
    C = [(0, 0), (1, 60), (2, 600), (5, 3600)]
    f = ev(C)
    ts = sorted({t for _, t in C})
    ttl = np.array([[t * 1000] * 5 for t in ts], np.uint32)
    hbm = int(0.05 * 10**9) // m.block_bytes
    cf = O.configs([[hbm, d * 10**9 // m.block_bytes, int(O.INF_CAP)] for d, _ in C], tuner=[ts.index(t) for _, t in C])
    f1 = ot.objective(m, cf, ot.replay(cf, ttl))            # O1 literal replay
    assert np.array_equal(f, f1)


def test_ttl_expansion_extension_mirrors_the_dram_rule():
    """R55 (extension, off by default): with latency falling in the TTL the way the DRAM test of
    Alg. 1 l.10-14 looks for, expand_ttl adds whole rows t_max + step over the initial DRAM range
    until the relative gain at the lowest DRAM row drops to tau_e; without it no TTL beyond the
    seed range is ever evaluated (R37)."""
    f = lambda t: 1.0 + 1e4 / (100.0 + t)                 # convex, decreasing latency in the TTL
    ev, _ = landscape(lambda d, t: f(t))                  # constant cost: no refinement
    p = S.SearchParams(0, 200, 100, 0, 200, 100, tau_e=0.05)
    log, _, _ = S.adaptive_search(ev, p)
    assert max(t for _, t, _ in log) == 200               # as written: the TTL axis never expands
    p = S.SearchParams(0, 200, 100, 0, 200, 100, tau_e=0.05, expand_ttl=True)
    log, _, trunc = S.adaptive_search(ev, p)
    tmax = max(t for _, t, _ in log)
    gain = lambda t: (f(t - 100) - f(t)) / f(t - 100)
    assert not trunc and tmax > 200 and gain(tmax) <= 0.05
    assert all(gain(t) > 0.05 for t in range(200, tmax, 100))
    for t in range(0, tmax + 1, 100):                      # every expansion adds the whole DRAM row
        assert {(0, t), (100, t), (200, t)} <= {(d, x) for d, x, _ in log}

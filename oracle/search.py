"""Oracle for row f1: Alg. 1 "Adaptive Pareto Exploration"
and the exact 3-D hypervolume the paper compares it with grid search by.

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never imports it.

Everything here is plain Python following the paper's steps in order; the readings of the
places the paper leaves open are DESIGN.md R36-R41:

  R36  Delta-latency / -throughput / -cost are relative: |a - b| / max(|a|, |b|, 1e-9).
  R37  "TTL = 0" in the DRAM-expansion step (Alg. 1 l.11-13) is the lowest TTL column t_min
       of the initial range (the paper's grids start at 0).  Expansion needs both
       (d_max - Delta_d, t_min) and (d_max, t_min) evaluated.
  R38  "adjacent pair" (Alg. 1 l.15): two evaluated points on one axis line (same t, or same d)
       with no evaluated point strictly between them.
  R39  midpoints are floor((d1+d2)/2) GB, floor((t1+t2)/2) s; a midpoint equal to an endpoint
       or to an evaluated point is dropped (termination).
  R40  each round evaluates the candidates in ascending (d, t) order; a round that would exceed
       the evaluation budget (or the round cap) is not started and the result is flagged
       truncated.
  R41  hypervolume: Lebesgue measure of the union of the boxes [p, ref] (minimisation), every
       point strictly better than ref in all three objectives.
"""
from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------- hypervolume
def area2d(xy, ref_xy) -> float:
    """Area of the union of the rectangles [x, rx] x [y, ry] (a staircase): sweep the points in
    ascending x (ties: ascending y); a point below the running minimum y adds the strip
    [x, rx] x [y, ymin)."""
    rx, ry = float(ref_xy[0]), float(ref_xy[1])
    pts = sorted((float(p[0]), float(p[1])) for p in xy)
    area, ymin = 0.0, ry
    for x, y in pts:
        if y < ymin:
            area += (rx - x) * (ymin - y)
            ymin = y
    return area


def hypervolume(points, ref) -> float:
    """Exact 3-D hypervolume by slicing along the third objective (HSO, While et al. 2006):
    with the points sorted by z, HV = sum_k A_k (z_{k+1} - z_k), z_{n+1} = ref_z, A_k = the
    2-D area dominated by the first k points (R41)."""
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    ref = np.asarray(ref, np.float64).reshape(3)
    for i, p in enumerate(pts):
        if not np.all(p < ref):
            raise ValueError(f"reference point not strictly worse than point {i}: {p.tolist()}")
    n = len(pts)
    if n == 0:
        return 0.0
    order = sorted(range(n), key=lambda i: pts[i, 2])
    hv = 0.0
    for k in range(n):
        z = pts[order[k], 2]
        z_next = ref[2] if k + 1 == n else pts[order[k + 1], 2]
        if z_next == z:
            continue
        hv += area2d(pts[order[:k + 1], :2], ref[:2]) * (z_next - z)
    return hv


# ---------------------------------------------------------------------------- Alg. 1
@dataclass
class SearchParams:
    d_min: int
    d_max: int
    d_step: int       # DRAM capacity axis, GB
    t_min: int
    t_max: int
    t_step: int       # disk TTL axis, s
    tau_e: float = 0.05
    tau_perf: float = 0.05
    tau_cost: float = 0.02
    max_evals: int = 1 << 20
    max_rounds: int = 0   # 0 = until C is empty
    expand_ttl: bool = False  # R55 (extension): also expand the TTL axis at the lowest DRAM row


def rel_delta(a: float, b: float) -> float:
    """R36."""
    return abs(a - b) / max(abs(a), abs(b), 1e-9)


def adjacent_pairs(S):
    """R38: consecutive evaluated points along each axis line."""
    by_t, by_d = defaultdict(list), defaultdict(list)
    for d, t in S:
        by_t[t].append(d)
        by_d[d].append(t)
    pairs = []
    for t, ds in by_t.items():
        ds.sort()
        pairs += [((ds[i], t), (ds[i + 1], t)) for i in range(len(ds) - 1)]
    for d, ts in by_d.items():
        ts.sort()
        pairs += [((d, ts[i]), (d, ts[i + 1])) for i in range(len(ts) - 1)]
    return pairs


def adaptive_search(evaluate, p: SearchParams):
    """Alg. 1.  `evaluate(list of (d, t)) -> array [n][3]` of (latency, -throughput,
    cost).  Returns (points [(d, t, round)], objectives [n][3], truncated)."""
    S = {}                                            # l.3: simulated configurations -> R
    log = []                                          # evaluation order (P in l.7)
    C = sorted({(d, t) for d in range(p.d_min, p.d_max + 1, p.d_step)    # l.2: uniform grid
                for t in range(p.t_min, p.t_max + 1, p.t_step)})
    rnd, truncated = 0, False
    while C:                                          # l.4 ... l.21 UNTIL C = empty
        if len(S) + len(C) > p.max_evals or (p.max_rounds and rnd >= p.max_rounds):
            truncated = True                          # R40
            break
        F = np.asarray(evaluate(C), np.float64).reshape(len(C), 3)
        for c, f in zip(C, F):                        # l.5-8: simulate every unvisited (d, t)
            S[c] = (float(f[0]), float(f[1]), float(f[2]))
            log.append((c[0], c[1], rnd))
        rnd += 1
        cand = set()                                  # l.9: C <- empty
        # l.10-14: DRAM expansion at the lowest TTL column (R37)
        col = [d for (d, t) in S if t == p.t_min]
        if col:
            dmax = max(col)
            lo = (dmax - p.d_step, p.t_min)
            if lo in S and rel_delta(S[lo][0], S[(dmax, p.t_min)][0]) > p.tau_e:
                for t in range(p.t_min, p.t_max + 1, p.t_step):
                    cand.add((dmax + p.d_step, t))
        # R55 (extension, not in Alg. 1): the l.10-14 test along the TTL axis at the lowest DRAM
        # row; the new row spans the initial DRAM range; TTLs stay below 2^32 ms
        if p.expand_ttl:
            row = [t for (d, t) in S if d == p.d_min]
            if row:
                tmax = max(row)
                lo = (p.d_min, tmax - p.t_step)
                if (tmax + p.t_step <= 0xFFFFFFFE // 1000 and lo in S
                        and rel_delta(S[lo][0], S[(p.d_min, tmax)][0]) > p.tau_e):
                    for d in range(p.d_min, p.d_max + 1, p.d_step):
                        cand.add((d, tmax + p.t_step))
        # l.15-19: refinement of adjacent pairs with a large performance and cost change
        for a, b in adjacent_pairs(S):
            fa, fb = S[a], S[b]
            if ((rel_delta(fa[0], fb[0]) > p.tau_perf or rel_delta(fa[1], fb[1]) > p.tau_perf)
                    and rel_delta(fa[2], fb[2]) > p.tau_cost):
                m = ((a[0] + b[0]) // 2, (a[1] + b[1]) // 2)   # R39
                if m != a and m != b:
                    cand.add(m)
        C = sorted(c for c in cand if c not in S)
    F = np.array([S[(d, t)] for d, t, _ in log], np.float64).reshape(-1, 3)
    return log, F, truncated


def grid_search(evaluate, d_range, t_range):
    """The paper's comparison: every cell of the uniform grid evaluated once."""
    C = sorted({(d, t) for d in range(*d_range) for t in range(*t_range)})
    return C, np.asarray(evaluate(C), np.float64).reshape(len(C), 3)


# ---------------------------------------------------------------------------- trace evaluator
def trace_evaluator(otrace, model, hbm_gb: float, block_bytes: int):
    """(d GB, t s) -> objectives through the oracle's own stack path (O2) and fluid model:
    HBM fixed at hbm_gb, DRAM d GB, TTL (lease) mode with a uniform disk TTL of t s;
    GB -> blocks = floor(GB * 1e9 / Bb) (R14)."""
    from oracle import oracle as O

    hbm = int(hbm_gb * 10**9) // block_bytes

    def evaluate(cands):
        ts = sorted({t for _, t in cands})
        tix = {t: i for i, t in enumerate(ts)}
        ttl = np.array([[t * 1000] * (otrace.K + 1) for t in ts], np.uint32).reshape(len(ts), otrace.K + 1)
        caps = [[hbm, d * 10**9 // block_bytes, int(O.INF_CAP)] for d, _ in cands]
        cf = O.configs(np.array(caps, np.uint64), policy=O.LRU, tuner=[tix[t] for _, t in cands])
        cnt = otrace.stack_counts(cf, ttl)
        return otrace.objective(model, cf, cnt)

    return evaluate

"""Oracle for row f2: Alg. 2 "ROI-Aware TTL Allocation"
over the group curves of P:748-756.

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never imports it.

Definitions, per group g with reuse intervals Delta_g (ms) and |B_g| unique blocks:
    H_g(t) = #{delta in Delta_g : delta <= t}
    C_g(t) = |B_g| t + sum_{delta in Delta_g} min(t, delta)          (block * ms)
Eq. 3: max sum_g H_g(t_g)  s.t.  sum_g C_g(t_g) <= B,  t >= 0.

Readings where the paper is silent or ill-posed (R43-R46):
  R43  ROI candidates (Alg. 2 l.4-5): TTLs are integer ms >= 1 (R_g(0) = H/0 is undefined).
       Between jumps H is flat and C grows, so the maximum of H/C sits at the left end of a flat
       piece: the candidates are {max(delta, 1) : delta in Delta_g}; argmax compared exactly
       (cross-multiplied integers), ties -> smallest t; an empty Delta_g -> 0.  (SPEC S:575's worked numbers 1/4 and 4/30 contradict the
       paper's C_g; this follows the paper: Delta = {1,3,3,7}, |B| = 2 gives 1/6, 3/16, 4/28.)
  R44  "SLSQP(max sum H s.t. sum C <= B, t >= 0) initialized at t_start" (l.15): H_g is a step
       function (zero gradient almost everywhere), so the local solve is an exact discrete local
       search over each group's jump points J_g = {0} u {distinct delta > 0}, started at t_start:
         (a) snap every t_g down to the largest jump point <= t_g (hits unchanged, cost lower);
         (b) while sum C > B: apply the down-move (g, t' < t_g in J_g) with the smallest lost
             hits per saved cost (H(t_g)-H(t'))/(C(t_g)-C(t')); ties -> smallest g, then largest t';
         (c) while an up-move (g, t' > t_g in J_g) fits the remaining budget: apply the one with
             the largest (H(t')-H(t_g))/(C(t')-C(t_g)); ties -> smallest g, then smallest t'.
  R45  perturbed starts (l.12-13): floor(Kp) = floor(sqrt(K)) starts,
       t_g = floor(t_init,g * (2^63 + u) / 2^64), u = fmix64(seed*1000003 + 64*s + g) (a factor
       in [0.5, 1.5)), s = 1..floor(sqrt(K)); non-negative by construction.
  R46  alpha = double(B) / double(sum_g C_g(t_roi,g)) (l.8-10); t_init,g = min(floor(alpha * t_roi,g),
       2^32 - 2); sum C(t_roi) = 0 -> t_init = 0.  The best start keeps the most hits (strictly
       more, l.17-20; t* = 0 if no start has a hit).
  R54  one more start, after the perturbed ones: the uniform TTL the paper compares against
       (one TTL for every group) at its largest feasible value
       t_u = max{t in [0, 2^32-2] : sum_g C_g(t) <= B} (C_g is non-decreasing in t, so a binary
       search).  The local solve never loses hits from a feasible start, so t* keeps at least
       the hits of the best uniform TTL at the same budget.
"""
from __future__ import annotations

import math

import numpy as np

from oracle.oracle import fmix64

M64 = (1 << 64) - 1
TTL_MAX = 0xFFFFFFFE


class Curve:
    """H_g, C_g of one group from its multiset Delta_g and |B_g|.  H and C follow the
    definitions literally; the tables HJ / CJ hold them at the jump points J (computed with the
    same two functions, once)."""

    def __init__(self, deltas, unique_blocks: int):
        d = sorted(int(x) for x in deltas)
        if any(x < 0 for x in d):
            raise ValueError("negative reuse interval")
        self.U = int(unique_blocks)
        self.N = len(d)
        self.d = d
        self._pre = [0]
        for x in d:
            self._pre.append(self._pre[-1] + x)
        # jump points: 0 and every distinct positive delta
        self.J = [0] + sorted({x for x in d if x > 0})
        self.HJ = [self.H(t) for t in self.J]
        self.CJ = [self.C(t) for t in self.J]

    def H(self, t: int) -> int:
        """#{delta <= t} (binary search in the sorted multiset)."""
        lo, hi = 0, self.N
        while lo < hi:
            m = (lo + hi) // 2
            if self.d[m] <= t:
                lo = m + 1
            else:
                hi = m
        return lo

    def C(self, t: int) -> int:
        """|B| t + sum min(t, delta): the deltas <= t contribute themselves, the others t."""
        h = self.H(t)
        return self.U * t + self._pre[h] + t * (self.N - h)

    def jump_index(self, t: int) -> int:
        """index of the largest jump point <= t."""
        lo, hi = 0, len(self.J)
        while lo < hi:
            m = (lo + hi) // 2
            if self.J[m] <= t:
                lo = m + 1
            else:
                hi = m
        return lo - 1


def curves_from_trace(export: dict, U_g, K: int):
    """Delta_g from the oracle trace export: every non-first access contributes its delta to the
    group of its request (groups R23)."""
    delta, req, grp = export["delta"], export["req"], export["group"]
    ok = (delta >= 0) & (delta < 0xFFFFFFFF)
    g_acc = grp[req]
    return [Curve(delta[ok & (g_acc == g)].tolist(), int(U_g[g])) for g in range(K + 1)]


def roi_ttl(c: Curve) -> int:
    """Alg. 2 l.4-5 with R43."""
    if c.N == 0:
        return 0
    best = None
    for t in sorted({max(x, 1) for x in c.d}):
        h, cc = c.H(t), c.C(t)
        if best is None or h * best[2] > best[1] * cc:
            best = (t, h, cc)
    return best[0]


def totals(curves, t):
    return sum(c.H(x) for c, x in zip(curves, t)), sum(c.C(x) for c, x in zip(curves, t))


def local_solve(curves, t_start, B: int):
    """R44 (a)-(c), on jump-point indices."""
    ix = [c.jump_index(x) for c, x in zip(curves, t_start)]             # (a) snap down
    hits = sum(c.HJ[i] for c, i in zip(curves, ix))
    cost = sum(c.CJ[i] for c, i in zip(curves, ix))
    while cost > B:                                                      # (b) restore feasibility
        best = None
        for g, c in enumerate(curves):
            hg, cg = c.HJ[ix[g]], c.CJ[ix[g]]
            for i in range(ix[g]):
                dh, dc = hg - c.HJ[i], cg - c.CJ[i]
                if dc <= 0:
                    continue
                if (best is None or dh * best[3] < best[2] * dc
                        or (dh * best[3] == best[2] * dc and g == best[0] and i > best[1])):
                    best = (g, i, dh, dc)
        if best is None:
            break
        g, i, dh, dc = best
        ix[g] = i
        hits, cost = hits - dh, cost - dc
    if cost > B:
        return [0] * len(curves)
    while True:                                                          # (c) ascend
        best = None
        for g, c in enumerate(curves):
            hg, cg = c.HJ[ix[g]], c.CJ[ix[g]]
            for i in range(ix[g] + 1, len(c.J)):
                dh, dc = c.HJ[i] - hg, c.CJ[i] - cg
                if dc <= 0 or dc > B - cost or dh <= 0:
                    continue
                if best is None or dh * best[3] > best[2] * dc:
                    best = (g, i, dh, dc)
        if best is None:
            break
        g, i, dh, dc = best
        ix[g] = i
        hits, cost = hits + dh, cost + dc
    return [c.J[i] for c, i in zip(curves, ix)]


def starts(t_init, K: int, seed: int = 0):
    """l.11-13 with R45."""
    P = [list(t_init)]
    for s in range(1, math.isqrt(K) + 1):
        row = []
        for g, x in enumerate(t_init):
            u = fmix64((seed * 1000003 + 64 * s + g) & M64)
            row.append((x * ((1 << 63) + u)) >> 64)
        P.append(row)
    return P


def uniform_ttl(curves, B: int) -> int:
    """R54: the largest t with sum_g C_g(t) <= B (binary search; C_g non-decreasing)."""
    lo, hi = 0, TTL_MAX
    while lo < hi:
        m = (lo + hi + 1) // 2
        if sum(c.C(m) for c in curves) <= B:
            lo = m
        else:
            hi = m - 1
    return lo


def allocate(curves, B: int, seed: int = 0):
    """Alg. 2.  Returns (t*, hits, cost, t_roi, t_init)."""
    K = len(curves) - 1
    t_roi = [roi_ttl(c) for c in curves]                                  # l.2-7
    c_unscaled = sum(c.C(x) for c, x in zip(curves, t_roi))              # l.8
    if c_unscaled > 0:
        alpha = float(B) / float(c_unscaled)                             # l.9 (fp64, R46)
        t_init = [min(int(math.floor(alpha * float(x))), TTL_MAX) for x in t_roi]   # l.10
    else:
        t_init = [0] * len(curves)
    best_t, best_hits, best_cost = [0] * len(curves), 0, 0               # l.14
    P = starts(t_init, K, seed) + [[uniform_ttl(curves, B)] * len(curves)]   # l.11-13 + R54
    for ts in P:                                                          # l.15-21
        sol = local_solve(curves, ts, B)
        h, c = totals(curves, sol)
        if h > best_hits:
            best_t, best_hits, best_cost = sol, h, c
    return best_t, best_hits, best_cost, t_roi, t_init

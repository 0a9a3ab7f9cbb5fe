"""Oracle for the trace analytics of row f4: X5 "Dynamic Storage Capacity" under the
oracle TTL and X6 reuse skew / Lorenz curve.

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never imports it.

Definitions (R47-R48), on the normalised trace (requests in arrival order, R6):
  X6  hits(b) = accesses of block b after its first ("reuse counts"); blocks sorted by hits
      descending; the Lorenz point i of n is the share of all hits held by the top
      k_i = ceil(i * U / (n - 1)) blocks; blocks_90 = the fewest top blocks holding >= 90% of the
      hits ("31.95% of blocks account for 90% of hits"), frac_90 = blocks_90 / U (no hits:
      frac_90 = 1, every Lorenz point 0).
  X5  after request r: cumulative(r) = distinct blocks seen in requests 0..r; active(r) = blocks
      seen in 0..r whose next access is in a later request (the oracle TTL keeps a block exactly
      until its next access and drops it after its last).
"""
from __future__ import annotations

import numpy as np


def block_hits(export: dict):
    """hits per distinct block (dict hash -> count of non-first accesses), plus the block count."""
    hits = {}
    for h, p in zip(export["hash"].tolist(), export["prev"].tolist()):
        if h not in hits:
            hits[h] = 0
        if p >= 0:
            hits[h] += 1
    return hits


def skew(export: dict, n_pts: int = 101):
    """X6: (total hits, blocks_90, frac_90, lorenz[n_pts], U)."""
    hits = sorted(block_hits(export).values(), reverse=True)
    U = len(hits)
    T = sum(hits)
    pre = [0]
    for x in hits:
        pre.append(pre[-1] + x)
    if T == 0:
        return 0, U, 1.0, [0.0] * n_pts, U
    k90 = next(k for k in range(1, U + 1) if 10 * pre[k] >= 9 * T)
    lor = []
    for i in range(n_pts):
        k = -(-i * U // (n_pts - 1))          # ceil(i U / (n - 1))
        lor.append(pre[k] / T)
    return T, k90, k90 / U, lor, U


def footprint(export: dict, R: int):
    """X5: cumulative[R], active[R] by direct per-request bookkeeping (next accesses found by a
    backward scan)."""
    h = export["hash"].tolist()
    req = export["req"].tolist()
    nxt_req = [None] * len(h)
    later = {}
    for j in range(len(h) - 1, -1, -1):                 # backward scan: next access of each position
        nxt_req[j] = later.get(h[j])
        later[h[j]] = req[j]
    by_req = [[] for _ in range(R)]
    for j, r in enumerate(req):
        by_req[r].append(j)
    seen, live = set(), {}
    cum, act = [], []
    for r in range(R):
        for j in by_req[r]:
            seen.add(h[j])
            if nxt_req[j] is not None:
                live[h[j]] = nxt_req[j]
            else:
                live.pop(h[j], None)
        cum.append(len(seen))
        act.append(len(live))
    return np.array(cum, np.int64), np.array(act, np.int64)

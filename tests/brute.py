"""O0: naive brute-force reference for TINY traces (pins the C oracle).

Independent of oracle/kareto_oracle.c: pure Python lists/dicts, victims found by a
full scan over the tier, LRU depths by an O(N^2) backward scan of the definition,
prev/delta by a linear scan.  Semantics: DESIGN.md "Replay semantics" (R9-R24),
which restate SURVEY 8.c.2 / PAPER P:357.
"""
from __future__ import annotations

INF = None


def touch_stream(chains_sorted):
    """chains_sorted: list of (arrival, group, [b_0..b_{n-1}]) in request order.
    Returns touch list [(req, k, block)] leaf->root per request, and s[r]."""
    touches, s = [], []
    for r, (_a, _g, ch) in enumerate(chains_sorted):
        s.append(len(touches))
        for k in range(len(ch) - 1, -1, -1):
            touches.append((r, k, ch[k]))
    s.append(len(touches))
    return touches, s


def prev_delta(chains_sorted):
    touches, s = touch_stream(chains_sorted)
    prev, delta = [], []
    for j, (r, _k, b) in enumerate(touches):
        p = -1
        for i in range(j - 1, -1, -1):
            if touches[i][2] == b:
                p = i
                break
        prev.append(p)
        delta.append(-1 if p < 0 else chains_sorted[r][0] - chains_sorted[touches[p][0]][0])
    return prev, delta


def lru_depths(chains_sorted):
    """d = 1-based LRU depth of the block at its request's start (None if first access),
    computed from the definition: 1 + #distinct other blocks touched since its last touch."""
    touches, s = touch_stream(chains_sorted)
    out = []
    for j, (r, k, b) in enumerate(touches):
        start = s[r]
        seen = set()
        found = False
        for i in range(start - 1, -1, -1):
            if touches[i][2] == b:
                found = True
                break
            seen.add(touches[i][2])
        out.append(len(seen) + 1 if found else None)
    return out


def replay(chains_sorted, cap, policy, tau):
    """Literal replay with naive structures.  cap = (c1, c2, c3) with c3 None = TTL mode;
    policy in {'lru','fifo','lfu'}; tau[g] ms (None = infinity)."""
    ttl_mode = cap[2] is None
    tier = {}        # block -> 1 HBM, 2 DRAM, 3 DISK
    last_t, last_seq, ins_seq, freq, lease_t = {}, {}, {}, {}, {}
    seen = set()
    gof = {}
    seq = 0
    c = dict(hit=[0, 0, 0], miss=0, evict=[0, 0, 0], disk_writes=0, hit_pos_sum=0, bytetime_block_ms=0,
             resident_after_hole=0)

    def key(b):
        if policy == "lru":
            return (last_seq[b],)
        if policy == "fifo":
            return (ins_seq[b],)
        return (freq[b], last_seq[b])

    def members(t):
        return [b for b, x in tier.items() if x == t]

    def capof(t):
        return cap[t - 1] if t < 3 else (0 if ttl_mode else cap[2])

    def cascade(t):
        nonlocal seq
        while len(members(t)) > capof(t):
            v = min(members(t), key=key)
            del tier[v]
            c["evict"][t - 1] += 1
            nxt = (t == 1) if ttl_mode else (t < 3)
            if nxt:
                seq += 1
                ins_seq[v] = seq
                tier[v] = t + 1
                cascade(t + 1)

    for (a, g, ch) in chains_sorted:
        for b in ch:
            gof[b] = g
        n = len(ch)
        if n == 0:
            continue
        if not ttl_mode:
            for b in list(members(3)):
                tg = tau[gof[b]]
                if tg is not None and a - last_t[b] > tg:
                    del tier[b]
        h = 0
        while h < n:
            b = ch[h]
            present = b in tier or (ttl_mode and b in seen and a - lease_t[b] <= tau[g])
            if not present:
                break
            h += 1
        for k in range(n):
            b = ch[k]
            if k < h:
                t = tier.get(b, 3)
                c["hit"][t - 1] += 1
                c["hit_pos_sum"] += k
            else:
                c["miss"] += 1
                if b in tier:
                    c["resident_after_hole"] += 1
            if ttl_mode and (b not in seen or a - lease_t[b] > tau[g]):
                c["disk_writes"] += 1
        for k in range(n - 1, -1, -1):
            b = ch[k]
            seq += 1
            if tier.get(b) == 1:
                if policy == "lru":
                    last_seq[b] = seq
                elif policy == "lfu":
                    freq[b] += 1
                    last_seq[b] = seq
            else:
                if b in tier:
                    del tier[b]
                    freq[b] += 1
                else:
                    freq[b] = 1
                last_seq[b] = seq
                ins_seq[b] = seq
                tier[b] = 1
                cascade(1)
            if ttl_mode and b in seen:
                c["bytetime_block_ms"] += min(a - lease_t[b], tau[g])
            last_t[b] = a
            lease_t[b] = a
            seen.add(b)
    if ttl_mode:
        for b in seen:
            c["bytetime_block_ms"] += tau[gof[b]]
        c["evict"][2] = 0
    else:
        c["disk_writes"] = c["evict"][1] if cap[2] > 0 else 0
        if any(t is not None for t in tau):
            c["evict"][2] = 0xFFFFFFFFFFFFFFFF
    return c


def hypervolume_cells(points, ref):
    """Brute-force 3-D hypervolume on the grid of all point coordinates: a cell is dominated
    iff some point is <= its lower corner in every coordinate (no sorting, no sweeping)."""
    axes = [sorted({float(p[a]) for p in points} | {float(ref[a])}) for a in range(3)]
    vol = 0.0
    for i in range(len(axes[0]) - 1):
        for j in range(len(axes[1]) - 1):
            for k in range(len(axes[2]) - 1):
                lo = (axes[0][i], axes[1][j], axes[2][k])
                if any(p[0] <= lo[0] and p[1] <= lo[1] and p[2] <= lo[2] for p in points):
                    vol += ((axes[0][i + 1] - axes[0][i]) * (axes[1][j + 1] - axes[1][j])
                            * (axes[2][k + 1] - axes[2][k]))
    return vol

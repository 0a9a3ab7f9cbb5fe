"""Oracle for row f3: queue-coupled disk prefetch and per-request TTFT
distributions (PAPER.md Obs. 2 and 4; user constraints such as a P99 TTFT bound,
P:510).

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never imports it.

Readings (R49-R53), for every configuration:
  R49  per request r (arrival order R6): the tiers serving its hit prefix in chain order, from the
       literal replay's lookup (O1, any policy).  For stack-eligible LRU configurations these are
       HBM blocks first, then DRAM, then disk, with h1 = #{d <= c1}, h2 = #{c1 < d <= c12},
       h3 = #{c12 < d <= C, delta <= tau} (CAPACITY) or #{d > c12, delta <= tau_g(r)} (TTL mode)
       from the pre-request depths d (first accesses never count) -- `per_request_hits`, a pin.
  R50  FCFS over I identical instances: r starts at s = max(a_r, min_i F_i) on the instance with
       the smallest free time (ties: lowest index); w_r = s - a_r; a_r = (arr_r - arr_0) * 1e-3 s.
  R51  disk prefetch: the prefix's disk blocks stream in chain order from arrival at bw_disk
       (= min(bw_max, bw_base + bw_slope * prov_GB), as the fluid model); the i-th one is loaded
       before service starts iff i <= x = (w_r * bw_disk) / Bb; the realised prefix ends at the
       first disk block not loaded, every later block is recomputed ("disk-based KV reloading
       exclusively during queuing time").  H, h2 = blocks / DRAM blocks of the realised
       prefix (LRU: H = h1 + h2 + min(h3, floor(x))).
  R52  service: prefill = (double)(P0_r - S) * 1e-12 with P0_r = alpha L + beta L(L-1)/2 and
       S = 16 alpha H + beta (256 H(H-1)/2 + 120 H) (R26); dram = (double)(h2 Bb) / bw_dram (R27);
       decode = (double)(dec o_r) * 1e-12; TTFT_r = (w_r + prefill) + dram; the instance is busy
       until ((s + prefill) + dram) + decode.
  R53  outputs: mean TTFT = 1e3 * (sum_r TTFT_r in arrival order) / R ms; P99 = 1e3 * the
       ceil(0.99 R)-th smallest TTFT (nearest rank); makespan M = max(span * 1e-3, max_i F_i);
       throughput = (Ltok + O) / M; disk hits capacity = sum h3, realized = sum h3'.
"""
from __future__ import annotations

import math

import numpy as np

INF32 = 0xFFFFFFFF


def request_arrays(trace):
    """Arrival (ms), input tokens L, output tokens o in the normalised order (stable by arrival,
    R6); L = token count (TOKENS mode) or input_tokens / 16 * blocks (HASHES mode)."""
    order = np.argsort(np.asarray(trace.arrival_ms, np.int64), kind="stable")
    off = np.asarray(trace.offsets, np.int64)
    cnt = off[1:] - off[:-1]
    if trace.tokens is not None:
        L = cnt
    else:
        L = np.asarray(trace.input_tokens, np.int64) if trace.input_tokens is not None else 16 * cnt
    return (np.asarray(trace.arrival_ms, np.int64)[order], L[order],
            np.asarray(trace.output_tokens, np.int64)[order])


def per_request_hits(d, delta, s, grp, cap, tau_row):
    """R49 for one configuration: lists h1, h2, h3 over requests."""
    c1, c2, c3 = cap
    ttl_mode = c3 == 0xFFFFFFFFFFFFFFFF
    c12 = c1 + c2
    C = c12 + (0 if ttl_mode else c3)
    H1, H2, H3 = [], [], []
    for r in range(len(s) - 1):
        tau = int(tau_row[grp[r]])
        h1 = h2 = h3 = 0
        for j in range(s[r], s[r + 1]):
            dj = int(d[j])
            if dj < 0:                                     # first access
                continue
            if dj <= c1:
                h1 += 1
            elif dj <= c12:
                h2 += 1
            elif (dj <= C or ttl_mode) and int(delta[j]) <= tau:
                h3 += 1
        H1.append(h1)
        H2.append(h2)
        H3.append(h3)
    return H1, H2, H3


def realised(prefix, x):
    """R51: (H, h2, disk blocks realised, disk blocks in the prefix) of a prefix tier sequence."""
    H = h2 = nd = real = 0
    open_ = True
    for t in prefix:
        if t == 3:
            nd += 1
            if open_ and float(nd) > x:
                open_ = False
        if open_:
            H += 1
            h2 += t == 2
            real += t == 3
    return H, h2, real, nd


def simulate(arr, L, o, prefixes, cfg_cap, medium, model, span_ms, Ltok, O):
    """R50-R53 for one configuration; prefixes[r] = tier sequence of request r's hit prefix.
    Returns dict(mean_ms, p99_ms, makespan_s, tok_per_s, disk_cap, disk_real, ttft [R] seconds)."""
    m = model
    bw_base, bw_slope, bw_max, _price = m.media[medium]
    ttl_mode = cfg_cap[2] == 0xFFFFFFFFFFFFFFFF
    Bb = m.block_bytes
    prov = m.ttl_prov_gb if ttl_mode else float((cfg_cap[2] * Bb) % (1 << 64)) / 1e9
    bw = min(bw_max, bw_base + bw_slope * prov)
    F = [0.0] * m.instances
    a0 = int(arr[0])
    total = 0.0
    ttft = []
    real = cap = 0
    M64 = (1 << 64) - 1
    for r in range(len(arr)):
        a = float(int(arr[r]) - a0) * 1e-3
        i = min(range(len(F)), key=lambda q: (F[q], q))
        start = max(a, F[i])
        w = start - a
        H, h2, rr, nd = realised(prefixes[r], (w * bw) / float(Bb))
        Lr = int(L[r])
        P0 = (m.alpha_ps * Lr + m.beta_ps * (Lr * (Lr - 1) // 2)) & M64
        S = (16 * m.alpha_ps * H + m.beta_ps * (256 * (H * (H - 1) // 2) + 120 * H)) & M64
        prefill = float((P0 - S) & M64) * 1e-12
        dram = float((h2 * Bb) & M64) / m.bw_dram
        decode = float((m.dec_ps * int(o[r])) & M64) * 1e-12
        t = (w + prefill) + dram
        ttft.append(t)
        total += t
        F[i] = ((start + prefill) + dram) + decode
        real += rr
        cap += nd
    R = len(arr)
    srt = sorted(ttft)
    k = -(-99 * R // 100)                                    # ceil(0.99 R)
    M = max(float(span_ms) * 1e-3, max(F))
    return dict(mean_ms=1e3 * (total / R), p99_ms=1e3 * srt[k - 1], makespan_s=M,
                tok_per_s=float(Ltok + O) / M, disk_cap=cap, disk_real=real, ttft=ttft)


def prefixes_from_lookup(lookup_tier, s):
    """per request, the hit prefix's tiers in chain order (block k sits at s_r + n_r - 1 - k)"""
    out = []
    for r in range(len(s) - 1):
        seq = []
        for j in range(s[r + 1] - 1, s[r] - 1, -1):
            if lookup_tier[j] == 0:
                break
            seq.append(int(lookup_tier[j]))
        out.append(seq)
    return out


def prefixes_from_counts(h1, h2, h3):
    """the LRU prefix shape: HBM blocks, then DRAM, then disk"""
    return [[1] * a + [2] * b + [3] * c for a, b, c in zip(h1, h2, h3)]


def evaluate(trace, otrace, cfgs, ttl, model):
    """R49-R53 for a list of configurations (oracle configs + TTL rows) on one trace; the hit
    prefixes come from the literal replay (O1) of each configuration."""
    e = otrace.export()
    arr, L, o = request_arrays(trace)
    s = e["s"].tolist()
    Ltok, O = int(L.sum()), int(o.sum())
    span = max(1, int(arr[-1]) - int(arr[0]))
    out = []
    for c in cfgs:
        cap = tuple(int(x) for x in c["cap"])
        _, lt = otrace.replay_lookup(c, ttl)
        out.append(simulate(arr, L, o, prefixes_from_lookup(lt.tolist(), s), cap, int(c["medium"]), model, span,
                            Ltok, O))
    return out

"""Oracle for row f3: queue-coupled disk prefetch and per-request TTFT
distributions (PAPER.md Obs. 2 and 4; user constraints such as a P99 TTFT bound,
P:510).

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never imports it.

Readings (R49-R53), for stack-eligible LRU configurations (section 5):
  R49  per request r (arrival order R6): prefix hits by tier from the pre-request LRU depths d and
       reuse intervals delta of its accesses: h1 = #{d <= c1}, h2 = #{c1 < d <= c12},
       h3 = #{c12 < d <= C, delta <= tau} (CAPACITY) or #{d > c12, delta <= tau_g(r)} (TTL mode);
       first accesses never count.  (Prefix closure: these are the tier sizes of the longest present
       prefix, HBM blocks first, then DRAM, then disk.)
  R50  FCFS over I identical instances: r starts at s = max(a_r, min_i F_i) on the instance with
       the smallest free time (ties: lowest index); w_r = s - a_r; a_r = (arr_r - arr_0) * 1e-3 s.
  R51  disk prefetch: the disk-resident prefix blocks stream from arrival at bw_disk
       (= min(bw_max, bw_base + bw_slope * prov_GB), as the fluid model); the ones loaded before
       service starts are hits, h3' = min(h3, floor((w_r * bw_disk) / Bb)); the hit prefix is
       H = h1 + h2 + h3' and every later block is recomputed ("disk-based KV reloading
       exclusively during queuing time").
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


def simulate(arr, L, o, h1, h2, h3, cfg_cap, medium, model, span_ms, Ltok, O):
    """R50-R53 for one configuration.  Returns dict(mean_ms, p99_ms, makespan_s, tok_per_s,
    disk_cap, disk_real, ttft [R] seconds)."""
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
        nload = math.floor((w * bw) / float(Bb))
        h3r = min(h3[r], nload)
        H = h1[r] + h2[r] + h3r
        Lr = int(L[r])
        P0 = (m.alpha_ps * Lr + m.beta_ps * (Lr * (Lr - 1) // 2)) & M64
        S = (16 * m.alpha_ps * H + m.beta_ps * (256 * (H * (H - 1) // 2) + 120 * H)) & M64
        prefill = float((P0 - S) & M64) * 1e-12
        dram = float((h2[r] * Bb) & M64) / m.bw_dram
        decode = float((m.dec_ps * int(o[r])) & M64) * 1e-12
        t = (w + prefill) + dram
        ttft.append(t)
        total += t
        F[i] = ((start + prefill) + dram) + decode
        real += h3r
        cap += h3[r]
    R = len(arr)
    srt = sorted(ttft)
    k = -(-99 * R // 100)                                    # ceil(0.99 R)
    M = max(float(span_ms) * 1e-3, max(F))
    return dict(mean_ms=1e3 * (total / R), p99_ms=1e3 * srt[k - 1], makespan_s=M,
                tok_per_s=float(Ltok + O) / M, disk_cap=cap, disk_real=real, ttft=ttft)


def evaluate(trace, otrace, cfgs, ttl, model):
    """All of R49-R53 for a list of configurations (oracle configs + TTL rows) on one trace."""
    e = otrace.export()
    d, _D = otrace.depth()
    arr, L, o = request_arrays(trace)
    s = e["s"].tolist()
    grp = e["group"].tolist()
    Ltok, O = int(L.sum()), int(o.sum())
    span = max(1, int(arr[-1]) - int(arr[0]))
    out = []
    for c in cfgs:
        cap = tuple(int(x) for x in c["cap"])
        row = ttl[int(c["tuner"])] if ttl is not None else [INF32] * (otrace.K + 1)
        h1, h2, h3 = per_request_hits(d, e["delta"], s, grp, cap, row)
        out.append(simulate(arr, L, o, h1, h2, h3, cap, int(c["medium"]), model, span, Ltok, O))
    return out

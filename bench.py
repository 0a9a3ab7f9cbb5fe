#!/usr/bin/env python
"""Benchmark of the Kareto configuration-evaluation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl kareto|reference]

A step = one pass of the whole hot path over the synthetic trace:
kareto_load_trace (ingest, K1 chain hash, K2 prev/delta/groups, K3 LRU depth) +
kareto_eval_grid_prepared (K4 histograms, K5+K7 counts+objective, allgather when N > 1) +
kareto_pareto_prepared (K8 prune + non-dominance), over the planner's configuration grid
prepared once (kareto_grid_create: validation, shard, device copies -- trace-independent).  The workload is BASELINE.json configs[1]
(default config 4, the north star's ">= 10^5-configuration grid on a 10^8-access trace"): a
G-agent trace of 1e8 block accesses (tokens 6.4 GB, larger than L2, so no flush is needed
between steps) and the 32 x 33 x 31 x 4-TTL capacity grid (130,944 configurations) with
diminishing-return pruning; `--config 2` is the 1M-request chat trace with the 32x32x16 LRU
grid (16,384 configurations), full Pareto frontier.

Multi-GPU (torchrun): one process per GPU; every rank loads the trace, evaluates its shard
of the grid, NCCL allgathers objective vectors; timing = max over ranks (strong scaling:
the grid is fixed).  `--impl reference` runs the oracle (plain CPU, oracle/) on the host
cores on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(kind="chat", R=10_000, grid=(4, 4, 4), div=(16, 4, 1), prune=None,
            desc="config1: G-chat 10k requests (~1.06M block accesses), 3-tier LRU 4x4x4 grid, fp64 model"),
    2: dict(kind="chat", R=1_000_000, grid=(32, 32, 16), div=(16, 2, 1), prune=None,
            desc="config2: G-chat 1M requests (~1.06e8 block accesses), 3-tier LRU 32x32x16 grid, full Pareto"),
    # config 3 down-scaled twin ("full O1 on a down-scaled twin (R = 10^4, same grid
    # shape)"): LRU/FIFO/LFU x 17 tuner rows (4 uniform, 7 quantile, 6 ROI), K = 16
    3: dict(kind="chat", R=10_000, grid="config3", prune=None, top_k=16,
            desc="config3 twin: G-chat 10k requests, A(16,U/16) x A(16,U/2) x (A(7,U) + TTL mode) x "
                 "{LRU,FIFO,LFU} x 17 tuner rows (103,680 configs, ~92K on the K6 replay)"),
    # config 4: agentic trace, 1e8 accesses, 70B-class blocks, GB grids of P:856 style, pruning on
    4: dict(kind="agent", N=100_000_000, grid="config4", prune=0.05, top_k=16,
            desc="config4: G-agent 1e8 block accesses, Bb = 5,242,880 B, HBM 0-1240 GB/40 x DRAM 0-4096 GB/128 x "
                 "disk 0-3600 GB/120 x uniform TTL {inf, 1h, 10min, 1min} (130,944 configs), pruning tau_e = 0.05"),
}


def tuner_rows_config3(delta_by_group, U_g, K):
    """17 tuner rows: 4 uniform, 7 nearest-rank quantiles of Delta_g, 6 ROI rows
    floor(a * t_roi), t_roi = argmax_delta H_g(delta)/C_g(delta) (Alg. 2 lines 4-5)."""
    inf = 0xFFFFFFFF
    rows = [[inf] * (K + 1), [3_600_000] * (K + 1), [600_000] * (K + 1), [60_000] * (K + 1)]
    for q in (0.5, 0.6, 0.7, 0.8, 0.9, 0.95, 0.99):
        row = []
        for g in range(K + 1):
            d = np.sort(delta_by_group[g])
            row.append(0 if len(d) == 0 else int(d[max(0, int(np.ceil(q * len(d))) - 1)]))
        rows.append(row)
    troi = []
    for g in range(K + 1):
        d = np.sort(delta_by_group[g]).astype(np.int64)
        if len(d) == 0:
            troi.append(0)
            continue
        vals = np.unique(np.maximum(d, 1))                               # candidates (DESIGN R43)
        H = np.searchsorted(d, vals, side="right")                       # #{delta <= t}
        csum = np.concatenate([[0], np.cumsum(d)])
        C = int(U_g[g]) * vals + csum[H] + vals * (len(d) - H)           # U_g t + sum min(t, delta)
        best = 0
        for i in range(1, len(vals)):                                    # exact cross-multiplied compare
            if int(H[i]) * int(C[best]) > int(H[best]) * int(C[i]):
                best = i
        troi.append(int(vals[best]))
    for a in (0.5, 1, 2, 4, 8, 16):
        rows.append([min(int(a * t), inf - 1) for t in troi])
    return np.array(rows, np.uint32)

# Algorithmic bytes per unit of each step of the path: K1 reads 64 B of tokens and
# writes the 8 B hash per block; K2 reads the 8 B hash and writes prev, delta, request and group
# fields (22 B per access); K3 reads (prev, request start) and writes the depth (12 B); K4 reads
# depth, D and delta (16 B); K6 touches 17 B of replay state per access and replayed configuration.
# The roofline of a pass credits it with its whole step's algorithmic bytes (a step's extra
# passes -- sort traffic, staging -- are overhead, not method bytes).
STEP_BYTES = {"K1": ("block", 72), "K2": ("access", 22), "K3": ("access", 12), "K4": ("access", 16),
              "K6": ("access-config", 17)}


def step_of(name: str):
    for k in ("K1", "K2", "K3", "K4", "K6"):
        if name.startswith(k):
            return k
    return None


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        # NVML in-process (the same counters nvidia-smi reports: clocks.sm, clocks.max.sm,
        # clocks_event_reasons.active); spawning nvidia-smi repeatedly stalls CUDA calls.  Opened
        # before the timed region, so a short region still gets its samples.
        self._nv, self._h = None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv, self._h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:
            pass

    def _sample(self):
        nv, h = self._nv, self._h
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((int(sm), int(mx), int(rs)))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.01)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sms = [s[0] for s in self.samples]
        reasons = set()
        for _, _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(reasons), "samples": len(self.samples)}


def grid_configs(K, U, grid, div):
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    m1, m2, m3 = grid
    c1, c2, c3 = A(m1, U // div[0]), A(m2, U // div[1]), A(m3, U // div[2])
    n = m1 * m2 * m3
    cfg = np.zeros(n, K.CONFIG_DTYPE)
    ii, jj, kk = np.meshgrid(np.arange(m1), np.arange(m2), np.arange(m3), indexing="ij")
    cfg["cap"][:, 0] = np.asarray(c1, np.uint64)[ii.ravel()]
    cfg["cap"][:, 1] = np.asarray(c2, np.uint64)[jj.ravel()]
    cfg["cap"][:, 2] = np.asarray(c3, np.uint64)[kk.ravel()]
    cfg["axis"] = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], 1)
    return cfg


def config3_grid(K, U, rows):
    """A(16,U/16) x A(16,U/2) x (A(7,U) + TTL mode) x 3 policies x rows,
    minus TTL mode with an all-infinite row (R22)."""
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    c1, c2, c3 = A(16, U // 16), A(16, U // 2), A(7, U)
    out = []
    for i, a in enumerate(c1):
        for j, b in enumerate(c2):
            for k in range(8):
                cap3 = c3[k] if k < 7 else K.INF
                for p in (K.LRU, K.FIFO, K.LFU):
                    for t in range(len(rows)):
                        if cap3 == K.INF and (rows[t] == 0xFFFFFFFF).any():
                            continue
                        out.append((a, b, cap3, p, t, i, j, k))
    cfg = np.zeros(len(out), K.CONFIG_DTYPE)
    arr = np.array(out, dtype=object)
    cfg["cap"] = np.array([[o[0], o[1], o[2]] for o in out], np.uint64)
    cfg["policy"] = [o[3] for o in out]
    cfg["tuner"] = [o[4] for o in out]
    cfg["axis"] = np.array([[o[5], o[6], o[7]] for o in out], np.int32)
    del arr
    return cfg


def config4_grid(K, block_bytes):
    """HBM 0-1240 GB step 40 x DRAM 0-4096 GB step 128 x disk 0-3600 GB step 120
    x uniform TTL {inf, 1 h, 10 min, 1 min}; GB -> blocks = floor(GB * 1e9 / Bb) (R14)."""
    gb = lambda lo, hi, step: np.arange(lo, hi + 1, step, dtype=np.uint64)
    h, d, s = gb(0, 1240, 40), gb(0, 4096, 128), gb(0, 3600, 120)
    blocks = lambda g: (g * np.uint64(10**9)) // np.uint64(block_bytes)
    ii, jj, kk, tt = np.meshgrid(np.arange(len(h)), np.arange(len(d)), np.arange(len(s)), np.arange(4), indexing="ij")
    cfg = np.zeros(ii.size, K.CONFIG_DTYPE)
    cfg["cap"][:, 0] = blocks(h)[ii.ravel()]
    cfg["cap"][:, 1] = blocks(d)[jj.ravel()]
    cfg["cap"][:, 2] = blocks(s)[kk.ravel()]
    cfg["tuner"] = tt.ravel()
    cfg["axis"] = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], 1)
    return cfg


def config4_rows(top_k):
    return np.array([[t] * (top_k + 1) for t in (0xFFFFFFFF, 3_600_000, 600_000, 60_000)], np.uint32)


def build_grid(K, spec, trace):
    """(configs, ttl rows or None) for a workload spec on a loaded trace."""
    g = spec["grid"]
    if g == "config3":
        delta = trace.export(K.X_DELTA)
        req = trace.export(K.X_REQ)
        grp = trace.export(K.X_GROUP)[req]
        ok = delta != 0xFFFFFFFF
        by_g = [delta[ok & (grp == gi)] for gi in range(trace.K + 1)]
        rows = tuner_rows_config3(by_g, trace.U_g, trace.K)
        return config3_grid(K, trace.U, rows), rows
    if g == "config4":
        return config4_grid(K, K.Model().block_bytes), config4_rows(trace.K)
    return grid_configs(K, trace.U, g, spec["div"]), None


def workload_config(spec, n_cfg, R, N, T):
    """The `config` object both arms print (identical keys and values for the same workload)."""
    return {"workload": spec["desc"], "n_configs": int(n_cfg), "n_requests": int(R), "n_accesses": int(N),
            "pruning": spec["prune"],
            "l2": f"no flush: each step's inputs ({T * 4 / 1e9:.1f} GB of tokens) exceed the 126 MB L2"}


def run_reference(args, spec):
    """Reference arm: the oracle (plain C, oracle/) as it stands, on the host cores.

    --full: one step over the full workload (the whole trace, every configuration; O2 Fenwick
    depths + stack closed forms for the LRU configurations, the fp64 model, R34 pruning and the
    O(n^2) dominance filter; configurations that need the literal replay O1 -- config 3 only --
    are sampled 48 at a time on every host thread and scaled in count, stated).
    Default: every step is the same pipeline over a SAMPLE trace of `--sample-requests` requests
    drawn from the same generator, with the full configuration grid; `ms_per_step` is the measured
    sample step, `value` scales its trace-proportional part linearly to the full trace (stated)."""
    import kareto_inputs as ki
    from oracle import oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2603_08739_b200 as K  # grid helpers / dtypes only (no device work)
    top_k = spec.get("top_k", 16)
    plan_full = ki.Plan(spec["kind"], R=spec.get("R", 0), N=spec.get("N", 0), seed=0)
    N_full, R_full = plan_full.n_blocks, plan_full.n_requests
    if args.full:
        tr = ki.synthetic(spec["kind"], R=spec.get("R", 0), N=spec.get("N", 0), seed=0)
    elif "R" in spec:
        tr = ki.synthetic(spec["kind"], R=min(spec["R"], args.sample_requests), seed=0)
    else:
        tr = ki.synthetic(spec["kind"], N=min(spec["N"], args.sample_requests * 100), seed=0)
    threads = os.cpu_count() or 1

    class _Shim:  # trace-like view of the oracle trace for build_grid
        def __init__(self, ot):
            e = ot.export()
            self.U, self.K, self.U_g = ot.U, ot.K, ot.U_g
            self._x = {K.X_DELTA: np.where(e["delta"] < 0, 0xFFFFFFFF, e["delta"]).astype(np.uint32),
                       K.X_REQ: e["req"].astype(np.uint32), K.X_GROUP: e["group"].astype(np.uint16)}

        def export(self, which):
            return self._x[which]

    def one():
        t0 = time.perf_counter()
        ot = O.OracleTrace(tr, top_k=top_k)
        kc, rows = build_grid(K, spec, _Shim(ot))
        cf = np.zeros(len(kc), O.CONFIG_DTYPE)
        for f in ("cap", "policy", "medium", "tuner", "axis"):
            cf[f] = kc[f]
        ttl = rows if rows is not None else np.full((1, top_k + 1), 0xFFFFFFFF, np.uint32)
        elig = np.array([ot.stack_eligible(cf[i:i + 1], ttl) for i in range(len(cf))], bool)
        cnt = np.zeros(len(cf), O.COUNTS_DTYPE)
        if elig.any():
            cnt[elig] = ot.stack_counts(cf[elig], ttl)
        t_trace = time.perf_counter() - t0
        # O1 replay: a stratified sample of the replay configurations, scaled in count
        rep = np.nonzero(~elig)[0]
        t_rep, n_samp = 0.0, 0
        if len(rep):
            samp = rep[np.linspace(0, len(rep) - 1, min(len(rep), 48)).astype(int)]
            n_samp = len(samp)
            t2 = time.perf_counter()
            cnt[samp] = ot.replay(cf[samp], ttl, threads=threads)
            t_rep = (time.perf_counter() - t2) * len(rep) / len(samp)
        t3 = time.perf_counter()
        fobj = ot.objective(O.Model(), cf, cnt, threads=threads)  # configurations across host threads
        t_obj = time.perf_counter() - t3  # the oracle's objective re-sums P0 over the requests: trace-proportional
        t4 = time.perf_counter()
        O.select(fobj, cf, spec["prune"], threads=threads)        # the O(n^2) rows on every host thread
        t_sel = time.perf_counter() - t4
        return t_trace, t_rep, t_sel, ot.N, len(cf), int(len(rep)), n_samp, t_obj, ot.R

    for _ in range(args.warmup):
        one()
    res = []
    w0 = time.perf_counter()
    for _ in range(args.steps):
        res.append(one())
    measured = (time.perf_counter() - w0) / max(1, args.steps)
    t_trace, t_rep, t_sel = (sum(r[i] for r in res) / len(res) for i in range(3))
    Ns, n, n_rep, n_samp = res[0][3], res[0][4], res[0][5], res[0][6]
    t_obj = sum(r[7] for r in res) / len(res)
    scale = N_full / Ns
    t_full = (t_trace + t_rep) * scale + t_obj * (R_full / res[0][8]) + t_sel
    t_sel += t_obj  # reported together below
    value = n / t_full
    if args.full:
        what = (f"full workload ({Ns} accesses, {n} configurations): oracle trace build + O2 Fenwick depths + "
                f"stack closed forms ({t_trace:.2f} s, sequential), fp64 model (configurations on {threads} threads) "
                f"+ pruning + O(n^2) dominance (rows on {threads} threads) ({t_sel:.2f} s)")
    else:
        what = (f"sample trace of {tr.n_requests} requests ({Ns} accesses, the same generator) with the full "
                f"{n}-configuration grid: oracle trace build + O2 depths + closed forms ({t_trace:.2f} s), fp64 model "
                f"+ pruning + O(n^2) dominance on {threads} threads ({t_sel:.2f} s); trace build, depths and replay "
                f"scaled x{scale:.1f} (accesses), the model x{R_full / res[0][8]:.1f} (requests) to the "
                f"full trace ({N_full} accesses): {t_full:.2f} s per full step")
    if n_rep:
        what += (f"; O1 literal replay of {n_samp} of the {n_rep} replay configurations on {threads} threads, "
                 f"scaled in count ({t_rep:.2f} s)")
    cores = threads  # the dominance rows (and config 3's O1 samples) run on every host thread
    line = {"impl": "reference", "metric": "configs evaluated/sec", "value": value, "unit": "configs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": measured * 1e3,
            "ms_per_full_step": t_full * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u64/f64", "data": "synthetic", "config": workload_config(spec, n, R_full, N_full, plan_full.n_tokens),
            "cpu_baseline": {"value": value, "unit": "configs/s", "cores": cores, "kind": "oracle", "sample": what},
            "e2e": {"value": value, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_search(args, K, ctx, tr, rank, spec, lengths):
    """Row f1 measurement, the P:856 protocol on a synthetic trace: grid search over DRAM
    0-4096 GB step 256 x disk TTL 0-3600 s step 120 (17 x 31 = 527 configurations, one batched
    kareto_eval_grid + kareto_pareto) against Alg. 1 seeded with DRAM 0-2048 GB step 512 x TTL
    0-2400 s step 600 (kareto_search); both frontiers' hypervolumes against one reference point
    strictly worse than every evaluated configuration (kareto_hypervolume).  HBM fixed, LRU,
    TTL (lease) mode with a uniform TTL; times are host wall clock around the synchronous calls
    with the trace resident, after one untimed run of each."""
    import torch
    # instance count from the no-cache work: I = max(1, round(busy_0 / (rho0 span))),
    # rho0 = 1.3 ("ins1-like", compute-constrained)
    m0 = K.Model()
    L = lengths.astype(np.int64)
    busy0 = (m0.alpha_ps * int(L.sum()) + m0.beta_ps * int((L * (L - 1) // 2).sum()) + m0.dec_ps * tr.O) * 1e-12
    inst = max(1, round(busy0 / (1.3 * tr.span_ms * 1e-3)))
    model = K.Model(instances=inst)
    Bb = model.block_bytes
    hbm = int(args.search_hbm_gb * 1e9) // Bb
    ds, ts = list(range(0, 4097, 256)), list(range(0, 3601, 120))
    cfg = np.zeros(len(ds) * len(ts), K.CONFIG_DTYPE)
    rows = np.array([[t * 1000] * (tr.K + 1) for t in ts], np.uint32)
    for a, d in enumerate(ds):
        for b, t in enumerate(ts):
            i = a * len(ts) + b
            cfg[i]["cap"] = (hbm, d * 10**9 // Bb, K.INF)
            cfg[i]["tuner"] = b
            cfg[i]["axis"] = (a, b, 0)

    def grid():
        _, obj = ctx.eval_grid(tr, cfg, model, rows)
        st, _ = ctx.pareto(obj, cfg, None)
        return obj, st

    def adaptive(expand_ttl=False):
        return ctx.search(tr, model, (0, 2048, 512), (0, 2400, 600), args.search_hbm_gb, expand_ttl=expand_ttl)

    grid(), adaptive()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    obj, st = grid()
    t_grid = time.perf_counter() - t0
    t0 = time.perf_counter()
    pts, trunc = adaptive()
    t_ad = time.perf_counter() - t0
    allf = np.vstack([obj, pts["obj"]])
    ref = allf.max(0) + np.abs(allf.max(0)) * 0.01 + 1e-12
    t0 = time.perf_counter()
    hv_g = ctx.hypervolume(obj, ref, mask=(st == 1).astype(np.uint8))
    t_hv = time.perf_counter() - t0
    hv_a = ctx.hypervolume(np.ascontiguousarray(pts["obj"]), ref, mask=(pts["status"] == 1).astype(np.uint8))
    # R55 (extension): Alg. 1 with the TTL axis expanded as well; its points may lie beyond the
    # grid's and the reference point above, so both frontiers are measured against a common one
    pts_x, trunc_x = adaptive(expand_ttl=True)
    allx = np.vstack([obj, pts["obj"], pts_x["obj"]])
    refx = allx.max(0) + np.abs(allx.max(0)) * 0.01 + 1e-12
    hv_gx = ctx.hypervolume(obj, refx, mask=(st == 1).astype(np.uint8))
    hv_ax = ctx.hypervolume(np.ascontiguousarray(pts_x["obj"]), refx, mask=(pts_x["status"] == 1).astype(np.uint8))
    if rank == 0:
        line = {"metric": "adaptive search (Alg. 1) vs grid search (P:856 protocol)", "unit": "evaluations",
                "grid_evals": int(len(cfg)), "adaptive_evals": int(len(pts)),
                "adaptive_rounds": int(pts["round"].max()) + 1 if len(pts) else 0, "truncated": bool(trunc),
                "hv_grid": hv_g, "hv_adaptive": hv_a, "hv_ratio": hv_a / hv_g if hv_g > 0 else None,
                "frontier_grid": int((st == 1).sum()), "frontier_adaptive": int((pts["status"] == 1).sum()),
                "grid_s": t_grid, "adaptive_s": t_ad, "hypervolume_s": t_hv, "reference_point": ref.tolist(),
                "ttl_expansion_R55": {"adaptive_evals": int(len(pts_x)), "truncated": bool(trunc_x),
                                      "max_ttl_s": int(pts_x["t_s"].max()) if len(pts_x) else None,
                                      "hv_ratio": hv_ax / hv_gx if hv_gx > 0 else None,
                                      "note": "extension, not Alg. 1 as written: the DRAM-expansion test also "
                                              "applied along the TTL axis at the lowest DRAM row"},
                "config": {"workload": spec["desc"], "n_accesses": tr.N, "hbm_gb": args.search_hbm_gb,
                           "instances": inst, "rho0": 1.3,
                           "policy": "LRU, TTL (lease) mode, uniform disk TTL", "block_bytes": Bb,
                           "grid": "DRAM 0-4096 GB step 256 x TTL 0-3600 s step 120",
                           "seed": "DRAM 0-2048 GB step 512 x TTL 0-2400 s step 600",
                           "thresholds": {"tau_e": 0.05, "tau_perf": 0.05, "tau_cost": 0.02}},
                "data": "synthetic", "timing": "host wall clock around synchronous ABI calls, trace resident"}
        print(json.dumps(line), flush=True)


def run_ttl(args, K, ctx, tr, rank, spec):
    """Row f2 measurement: Alg. 2 (kareto_ttl_allocate) on the config's trace at budgets of 1%, 5%
    and 20% of the cost of leasing every block for the whole span, against the best uniform TTL
    with the same budget (bisection over kareto_ttl_eval batches).  Host wall clock around the
    synchronous calls, trace resident, after one untimed run."""
    import time as _t
    G = tr.K + 1
    span = int(tr.span_ms)
    _, full = ctx.ttl_eval(tr, np.full((1, G), span, np.uint32))
    full = int(full[0])
    ctx.ttl_roi(tr)
    t0 = _t.perf_counter()
    t_roi, h_roi, c_roi = ctx.ttl_roi(tr)
    t_roi_s = _t.perf_counter() - t0
    total_reuse = int(tr.reuse_g.sum())
    rows = []
    for frac in (0.01, 0.05, 0.2):
        B = int(frac * full)
        ctx.ttl_allocate(tr, B, seed=0)
        t0 = _t.perf_counter()
        r = ctx.ttl_allocate(tr, B, seed=0)
        t_alloc = _t.perf_counter() - t0
        lo, hi = 0, span                        # best uniform TTL within the budget
        while lo < hi:
            cand = np.linspace(lo, hi, 65).astype(np.int64)
            hh, cc = ctx.ttl_eval(tr, np.repeat(cand[:, None], G, 1).astype(np.uint32))
            ok = cand[cc <= B]
            new_lo = int(ok.max()) if len(ok) else lo
            bad = cand[cc > B]
            new_hi = int(bad.min()) - 1 if len(bad) else hi
            if (new_lo, new_hi) == (lo, hi):
                break
            lo, hi = new_lo, max(new_lo, new_hi)
        hu, cu = ctx.ttl_eval(tr, np.full((1, G), lo, np.uint32))
        rows.append({"budget_frac": frac, "budget_block_ms": B, "alg2_hits": r["hits"], "alg2_cost": r["cost"],
                     "alg2_s": t_alloc, "uniform_ttl_ms": lo, "uniform_hits": int(hu[0]), "uniform_cost": int(cu[0]),
                     "hit_gain_vs_uniform": r["hits"] / max(1, int(hu[0])), "t_ms": r["t"].tolist()})
    if rank == 0:
        line = {"metric": "Alg. 2 group-TTL allocation (row f2)", "unit": "hits", "groups": G,
                "total_reuse_events": total_reuse, "full_lease_cost_block_ms": full, "roi_s": t_roi_s,
                "t_roi_ms": t_roi.tolist(), "budgets": rows,
                "config": {"workload": spec["desc"], "n_accesses": tr.N, "top_k": tr.K},
                "data": "synthetic", "timing": "host wall clock around synchronous ABI calls, trace resident"}
        print(json.dumps(line), flush=True)


def run_queue(args, K, ctx, tr, rank, spec, lengths):
    """Row f3 measurement (Obs. 2 / Obs. 4): a 4 x 8 x 8 LRU grid (HBM A(4, U/16) x DRAM
    A(8, U/2) x disk A(8, U), CAPACITY, no TTL) through kareto_eval_queue at a low (rho0 = 0.3,
    "ins4-like") and a high (rho0 = 1.3, "ins1-like") workload density, I = max(1, round(busy_0 /
    (rho0 span))); reports the realised share of the capacity-predicted disk hits, TTFT, the
    configurations meeting P99 TTFT <= 2 s, and the device time per configuration."""
    import torch
    m0 = K.Model()
    L = lengths.astype(np.int64)
    busy0 = (m0.alpha_ps * int(L.sum()) + m0.beta_ps * int((L * (L - 1) // 2).sum()) + m0.dec_ps * tr.O) * 1e-12
    U = tr.U
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps = [[a, b, c] for a in A(4, U // 16) for b in A(8, U // 2) for c in A(8, U)]
    cfg = K.configs(caps)
    res = []
    for rho in (0.3, 1.3):
        inst = max(1, round(busy0 / (rho * tr.span_ms * 1e-3)))
        model = K.Model(instances=inst)
        ctx.eval_queue(tr, cfg[:2], model)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q = ctx.eval_queue(tr, cfg, model)
        dt = time.perf_counter() - t0
        _, obj = ctx.eval_grid(tr, cfg, model)
        ok = q["ttft_p99_ms"] <= 2000.0
        f = obj.copy()
        f[:, 0] = q["ttft_mean_ms"]
        f[:, 1] = -q["tokens_per_s"]
        front = 0
        if ok.any():
            st, front = ctx.pareto(np.ascontiguousarray(f[ok]), None, None)
        capd = int(q["disk_hits_capacity"].sum())
        real = int(q["disk_hits_realized"].sum())
        res.append({"rho0": rho, "instances": inst, "configs": len(cfg), "seconds": dt,
                    "configs_per_s": len(cfg) / dt,
                    "disk_hits_capacity": capd, "disk_hits_realized": real,
                    "realized_fraction": real / capd if capd else None,
                    "ttft_mean_ms_range": [float(q["ttft_mean_ms"].min()), float(q["ttft_mean_ms"].max())],
                    "ttft_p99_ms_range": [float(q["ttft_p99_ms"].min()), float(q["ttft_p99_ms"].max())],
                    "fluid_mean_ttft_ms_range": [float(obj[:, 0].min()), float(obj[:, 0].max())],
                    "p99_le_2s": int(ok.sum()), "frontier_under_p99": int(front)})
    if rank == 0:
        print(json.dumps({"metric": "queue-coupled disk prefetch (row f3)", "unit": "configs/s",
                          "densities": res, "config": {"workload": spec["desc"], "n_accesses": tr.N,
                                                        "n_requests": tr.R, "grid": "A(4,U/16) x A(8,U/2) x A(8,U), LRU"},
                          "data": "synthetic", "timing": "host wall clock around the synchronous call"}), flush=True)


def run_emulate(args, K, spec, cfg, ttl, model, dev_inputs, top_k, stream, N, U, n_cfg):
    """Row f4 on one GPU: W loopback ranks (one host thread + CUDA stream each) run the
    time-sharded step (load_trace_sharded + eval_grid + pareto); the W shards' kernels and the
    loopback exchanges share the one GPU, so the step time measures the TOTAL device work of the
    sharded algorithm (its work efficiency against the unsharded step), not multi-GPU speed."""
    import torch
    W = args.emulate_ranks
    arr_d, out_d, off_d, tok_d = dev_inputs
    ctx1 = K.Context(torch.cuda.current_device(), stream.cuda_stream)

    def step1():
        t = ctx1.load_trace(arr_d, out_d, off_d, tokens=tok_d, top_k=top_k)
        _, o = ctx1.eval_grid(t, cfg, model, ttl)
        ctx1.pareto(o, cfg, spec["prune"])
        t.free()

    for _ in range(args.warmup):
        step1()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step1()
    torch.cuda.synchronize()
    ms1 = (time.perf_counter() - t0) * 1e3 / args.steps

    group = K.Loopback(W)
    barrier = threading.Barrier(W)
    times, err, shard = [[] for _ in range(W)], [None] * W, [None] * W

    def body(r):
        try:
            torch.cuda.set_device(stream.device)
            s = torch.cuda.Stream()
            c = K.Context(torch.cuda.current_device(), s.cuda_stream, loopback=group, rank=r)

            def stepw():
                t = c.load_trace(arr_d, out_d, off_d, tokens=tok_d, top_k=top_k, time_shard=True)
                _, o = c.eval_grid(t, cfg, model, ttl)
                c.pareto(o, cfg, spec["prune"])
                shard[r] = t.pos_hi - t.pos_lo
                t.free()

            for _ in range(args.warmup):
                stepw()
            for _ in range(args.steps):  # per step: all ranks start together, each times its own end
                barrier.wait()
                torch.cuda.synchronize()
                barrier.wait()
                a = time.perf_counter()
                stepw()
                torch.cuda.synchronize()
                times[r].append((time.perf_counter() - a) * 1e3)
            barrier.wait()
            c.close()
        except BaseException as e:  # noqa: BLE001
            err[r] = e
            barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    msW = statistics.median(max(times[r][i] for r in range(W)) for i in range(args.steps))
    print(json.dumps({"metric": "time-sharded step, all shards on one GPU (row f4 work efficiency)",
                      "value": msW, "unit": "ms", "emulated_ranks": W, "unsharded_ms_per_step": ms1,
                      "work_ratio": msW / ms1, "shard_accesses": shard, "n_accesses": N, "n_unique": U,
                      "n_configs": n_cfg, "steps": args.steps, "warmup": args.warmup,
                      "config": {"workload": spec["desc"]}, "data": "synthetic",
                      "timing": "median over steps of the slowest rank's host wall clock (steps started "
                                "together); the W ranks' kernels and the loopback exchanges (device-to-device "
                                "copies) share the one GPU, host-thread scheduling makes single steps noisy"}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="kareto", choices=["kareto", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full", type=int, default=1,
                    help="cpu_baseline: 1 = one full-workload oracle step (default), 0 = scaled sample")
    ap.add_argument("--sample-requests", type=int, default=50_000,
                    help="reference arm: requests of the sample trace each step processes")
    ap.add_argument("--full", action="store_true",
                    help="reference arm: one step over the FULL workload (no sample, no extrapolation)")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no cpu baseline / e2e)")
    ap.add_argument("--search", action="store_true",
                    help="row f1: Alg. 1 adaptive search vs the P:856 grid search on the config's trace")
    ap.add_argument("--search-hbm-gb", type=float, default=320.0)
    ap.add_argument("--queue", action="store_true",
                    help="row f3: queue-coupled disk prefetch at low and high workload density (Obs. 2/4)")
    ap.add_argument("--analytics", action="store_true",
                    help="row f4 analytics: X6 reuse skew and X5 oracle-TTL footprint of the config's trace")
    ap.add_argument("--ttl", action="store_true",
                    help="row f2: Alg. 2 group-TTL allocation vs the best uniform TTL on the config's trace")
    ap.add_argument("--time-shard", default="auto", choices=["auto", "on", "off"],
                    help="row f4: split the trace passes by time across ranks (auto: when world > 1 and the "
                         "grid is all stack-path configurations)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="row f4 on ONE GPU: W loopback ranks (threads) run the time-sharded step; reports the "
                         "total device work of all shards against the unsharded step")
    args = ap.parse_args()
    spec = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, spec)
        return

    import torch
    import torch.distributed as dist

    import kareto_inputs as ki
    import paper_2603_08739_b200 as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    from paper_2603_08739_b200 import dist as kd
    ctx = kd.create_context(local, stream.cuda_stream)
    top_k = spec.get("top_k", 16)

    # ---- synthetic workload (seeded; host pinned buffers, then device copies)
    t0 = time.time()
    plan = ki.Plan(spec["kind"], R=spec.get("R", 0), N=spec.get("N", 0), seed=0)
    R, T = plan.n_requests, plan.n_tokens
    arr_h = torch.empty(R, dtype=torch.int64, pin_memory=True)
    out_h = torch.empty(R, dtype=torch.int32, pin_memory=True)
    off_h = torch.empty(R + 1, dtype=torch.int64, pin_memory=True)
    tok_h = torch.empty(T, dtype=torch.int32, pin_memory=True)
    plan.fill_meta(arr_h.numpy(), out_h.numpy(), off_h.numpy())
    plan.fill_tokens_ptr(tok_h.data_ptr())
    gen_s = time.time() - t0
    with torch.cuda.stream(stream):
        arr_d, out_d, off_d, tok_d = (x.to(f"cuda:{local}", non_blocking=True) for x in (arr_h, out_h, off_h, tok_h))
    stream.synchronize()

    def load_dev(time_shard=False):
        return ctx.load_trace(arr_d, out_d, off_d, tokens=tok_d, top_k=top_k, time_shard=time_shard)

    if args.search:
        run_search(args, K, ctx, load_dev(), rank, spec, np.diff(off_h.numpy()))
        return
    if args.ttl:
        run_ttl(args, K, ctx, load_dev(), rank, spec)
        return
    if args.queue:
        run_queue(args, K, ctx, load_dev(), rank, spec, np.diff(off_h.numpy()))
        return
    if args.analytics:
        tr = load_dev()
        ctx.analytics(tr, series=False)
        t0 = time.perf_counter()
        a = ctx.analytics(tr, n_pts=11, series=False)
        dt = time.perf_counter() - t0
        if rank == 0:
            print(json.dumps({"metric": "trace analytics X5/X6 (row f4)", "unit": "s", "value": dt,
                              "unique_blocks": a["unique_blocks"], "total_hits": a["total_hits"],
                              "frac_blocks_for_90pct_hits": a["frac_90"], "lorenz_deciles": a["lorenz"].tolist(),
                              "peak_active_blocks": a["peak_active"], "final_cumulative_blocks": a["final_cumulative"],
                              "config": {"workload": spec["desc"], "n_accesses": tr.N},
                              "data": "synthetic", "timing": "host wall clock around the synchronous call"}),
                  flush=True)
        return

    tr = load_dev()
    N, U = tr.N, tr.U
    cfg, ttl = build_grid(K, spec, tr)   # the planner's grid (not part of the timed hot path)
    n_cfg = len(cfg)
    if ttl is None:
        n_replay = int((cfg["policy"] != K.LRU).sum())
    else:
        nonuni = (ttl[cfg["tuner"]] != ttl[cfg["tuner"]][:, :1]).any(1)
        n_replay = int(((cfg["policy"] != K.LRU) | ((cfg["cap"][:, 2] != K.INF) & nonuni)).sum())
    model = K.Model()
    if args.emulate_ranks > 0:
        tr.free()
        run_emulate(args, K, spec, cfg, ttl, model, (arr_d, out_d, off_d, tok_d), top_k, stream, N, U, n_cfg)
        return
    tshard = args.time_shard == "on" or (args.time_shard == "auto" and world > 1 and n_replay == 0)
    n_local = N
    if tshard:  # this rank's slice of the accesses (the units its trace passes process)
        tr.free()
        tr = load_dev(True)
        n_local = tr.pos_hi - tr.pos_lo
    req_lo, req_hi = tr.req_lo, tr.req_hi
    cnt_d = torch.empty((n_cfg, 11), dtype=torch.int64, device=f"cuda:{local}")
    obj_d = torch.empty((n_cfg, 3), dtype=torch.float64, device=f"cuda:{local}")
    st_d = torch.empty(n_cfg, dtype=torch.uint8, device=f"cuda:{local}")
    tr.free()
    # the planner's grid, prepared once (kareto_grid_create: validation, shard, split, device copies);
    # every step evaluates it against a freshly loaded trace
    grid = ctx.grid(cfg, ttl, n_groups=top_k + 1)

    def step():
        t = load_dev(tshard)
        ctx.eval_prepared(t, grid, model, counts=cnt_d, obj=obj_d)
        _, nf = ctx.pareto_prepared(obj_d, grid, spec["prune"], status=st_d)
        t.free()
        return nf

    for _ in range(args.warmup):
        nf = step()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: device time with CUDA events on the library stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_counter()
    barrier()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            nf = step()
        ev1.record(stream)
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = ctx.launch_counter() - l0
    t = torch.tensor([ms_total], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = n_cfg / (ms_step * 1e-3)

    # ---- per-pass device times (profiled replay of the same steps) for the roofline
    ctx.set_profiling(True)
    ctx.pass_times(reset=True)
    prof_steps = 1 if ms_step > 10_000 else max(3, min(args.steps, 10))
    for _ in range(prof_steps):
        step()
    passes = ctx.pass_times(reset=True)
    ctx.set_profiling(False)
    peak, peak_src = measured_peak()
    units = {"block": n_local, "access": n_local}
    k6 = [p for p in passes if p["name"].startswith("K6_replay")]
    if k6:  # one roofline entry for the replay (its class passes merged)
        passes = [p for p in passes if not p["name"].startswith("K6_replay")] + [
            {"name": "K6_replay", "ms": sum(p["ms"] for p in k6), "launches": sum(p["launches"] for p in k6),
             "own": 1}] + [dict(p, name=p["name"].replace("K6_replay", "K6class")) for p in k6
                           if p["name"] != "K6_replay"]  # per-class passes (sequential replay) only
    if k6 and n_replay:
        # this rank's replayed configurations (the cost-weighted shard is ~1/world of them) over all
        # K6 launches (waves of the four classes)
        units["access-config"] = N * n_replay / world * prof_steps / sum(p["launches"] for p in k6)
    roof = None
    # the dominant pass of the step by device time, own kernel or library call alike (CUB sorts
    # included), credited with its step's algorithmic bytes (STEP_BYTES)
    ranked = sorted((p for p in passes if step_of(p["name"]) and p["launches"] > 0), key=lambda p: -p["ms"])
    if ranked:
        top = ranked[0]
        stp = step_of(top["name"])
        unit, bpu = STEP_BYTES[stp]
        per_launch_ms = top["ms"] / top["launches"]
        algo_bytes = bpu * units[unit] if unit != "access-config" else bpu * units[unit]
        achieved = algo_bytes / (per_launch_ms * 1e-3) / 1e9
        step_ms = sum(p["ms"] for p in passes if step_of(p["name"]) == stp) / prof_steps
        step_bytes = bpu * units[unit] * (top["launches"] / prof_steps)
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", f"ncu_traffic_config{args.config}.json")
        if os.path.exists(tp):  # DRAM bytes per launch from a committed `ncu --set full` capture
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj.get("dram_bytes_per_launch", {}).get(top["name"])
            traffic_src = tj.get("source") if traffic is not None else None
        roof = {"kernel": top["name"], "own": bool(top["own"]), "bound": "hbm", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": peak_src, "algorithmic_bytes_per_launch": algo_bytes, "bytes_per_unit": bpu,
                "unit_of_work": unit, "step": stp, "avg_launch_ms": per_launch_ms,
                "share_of_step": top["ms"] / prof_steps / ms_step,
                "step_frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak if step_ms > 0 else None,
                "runner_up": [{"kernel": p["name"], "ms": round(p["ms"] / prof_steps, 4)} for p in ranked[1:4]]}
    stage_ms = {p["name"]: round(p["ms"] / prof_steps, 4) for p in passes}
    # end-to-end algorithmic roofline: the bytes the method itself must move
    # per step -- K1 72 B/block (64 B tokens + 8 B hash), K2 22 B/access, K3 12 B/access, K4
    # 16 B/access, K6 17 B per replayed access-config -- over (step time x measured HBM peak)
    algo_step = 122 * n_local + 17 * n_local * n_replay / world
    algo_roof = {"bytes_per_step": algo_step, "frac": algo_step / (ms_step * 1e-3) / (peak * 1e9),
                 "per_unit": "K1 72 B/block + K2 22 + K3 12 + K4 16 B/access (+ K6 17 B/access-config)"}

    # ---- end to end through the C ABI with host (pinned) buffers, H2D + D2H in the region
    e2e = None
    if not args.profile_only and args.e2e_steps > 0:
        cnt_h = np.zeros(n_cfg, K.COUNTS_DTYPE)
        obj_h = np.zeros((n_cfg, 3), np.float64)
        arr_np, out_np, off_np, tok_np = arr_h.numpy(), out_h.numpy(), off_h.numpy(), tok_h.numpy().view(np.uint32)

        def step_host():
            t_ = ctx.load_trace(arr_np, out_np, off_np, tokens=tok_np, top_k=top_k, time_shard=tshard)
            ctx.eval_prepared(t_, grid, model, counts=cnt_h, obj=obj_h)
            s_, _ = ctx.pareto_prepared(obj_h, grid, spec["prune"])
            t_.free()
            return s_

        step_host()
        barrier()
        w0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            step_host()
        e1.record(stream)
        barrier()
        wall = (time.perf_counter() - w0) / args.e2e_steps
        te = torch.tensor([wall], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        wall = float(te.item())
        # a time-sharded rank copies only the token range covering its requests (as the library does)
        tok_bytes = tok_np.nbytes
        if tshard:
            sel = np.argsort(arr_np, kind="stable")[req_lo:req_hi]
            o0 = off_np[sel]
            o1 = o0 + 16 * ((off_np[sel + 1] - o0) // 16)
            m = o1 > o0
            tok_bytes = 4 * int(o1[m].max() - o0[m].min()) if m.any() else 0
        h2d = arr_np.nbytes + out_np.nbytes + off_np.nbytes + tok_bytes + 24 * n_cfg  # + obj for K8 (host)
        d2h = cnt_h.nbytes + obj_h.nbytes + n_cfg
        e2e = {"value": n_cfg / wall, "unit": "configs/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": wall * 1e3,
               "timing": "host wall clock around synchronous ABI calls (inputs in pinned host memory)"}

    # ---- oracle on host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        try:
            r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                                "--warmup", "0", "--config", str(args.config), "--sample-requests",
                                str(args.sample_requests)] + (["--full"] if args.cpu_full else []),
                               capture_output=True, text=True, timeout=1800)
            ref = json.loads(r.stdout.strip().splitlines()[-1])
            cpu = ref["cpu_baseline"]
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "configs/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": "configs evaluated/sec", "value": value, "unit": "configs/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
                "config": workload_config(spec, n_cfg, R, N, T),
                "workload_detail": {"n_unique": U, "tokens_bytes": int(T * 4),
                                    "parallelism": (f"time-shard x{world} (trace passes split by time: owner exchange "
                                                    f"of first/last accesses, boundary LRU sets, histogram allreduce)"
                                                    if tshard else f"config-shard x{world} (trace passes replicated)"),
                                    "replay_configs": n_replay},
                "block_accesses_per_s": N / (ms_step * 1e-3),
                "effective_access_configs_per_s": N * n_cfg / (ms_step * 1e-3),
                "frontier": nf, "roofline": roof, "algorithmic_roofline": algo_roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches),
                "gpu_launches_per_step": launches / args.steps, "clocks": clk.summary(), "stage_ms": stage_ms,
                "generation_s": round(gen_s, 2)}
        print(json.dumps(line), flush=True)
    grid.free()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Full-size config 3 on a sample (row a7): the K6 replay on the R = 1e6 chat trace (1.06e8
accesses, U = 2.27e7, K = 16) for a stratified sample of the 103,680-configuration grid, timed on
the GPU and compared with the oracle's O1 literal replay, counts bit-exact.

The tuner rows come from the ORACLE's trace export (as in tests/test_gpu_fullsize.py); the grid is
bench.py's config-3 definition at full size.  Prints one JSON line: the sample, GPU seconds,
access-configurations per second, the O1 comparison and the extrapolated time of the whole grid's
replay configurations at the measured rate.

    python tools/config3_fullsize_sample.py --per-cell 12
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=1_000_000)
    ap.add_argument("--per-cell", type=int, default=12, help="configurations per (policy, disk mode) replay cell")
    ap.add_argument("--oracle-threads", type=int, default=0)
    ap.add_argument("--ttl-groups", type=int, default=0,
                    help="instead of the stratified sample: every TTL row of this many (c1, c2) groups for FIFO "
                         "and LFU in TTL mode (the collapsed path, forced with KARETO_K6_COLLAPSE)")
    ap.add_argument("--oracle-sample", type=int, default=0, help="O1 on only this many of the sampled configurations")
    args = ap.parse_args()
    import torch

    import bench
    import kareto_inputs as ki
    import paper_2603_08739_b200 as K
    from oracle import oracle as O

    spec = bench.CONFIGS[3]
    t0 = time.time()
    tr = ki.synthetic(spec["kind"], R=args.requests, seed=0)
    ot = O.OracleTrace(tr, top_k=spec["top_k"])
    e = ot.export()
    ok = (e["delta"] >= 0) & (e["delta"] < 0xFFFFFFFF)
    g_acc = e["group"][e["req"]]
    by_g = [e["delta"][ok & (g_acc == g)] for g in range(spec["top_k"] + 1)]
    rows = bench.tuner_rows_config3(by_g, ot.U_g, spec["top_k"])
    del e, ok, g_acc, by_g
    cfg = bench.config3_grid(K, ot.U, rows)
    prep_s = time.time() - t0
    ttl_mode = cfg["cap"][:, 2] == np.uint64(0xFFFFFFFFFFFFFFFF)
    nonuni = (rows[cfg["tuner"]] != rows[cfg["tuner"]][:, :1]).any(1)
    replay = (cfg["policy"] != K.LRU) | (~ttl_mode & nonuni)
    rng = np.random.default_rng(5)
    idx, cells = [], {}
    for p, pn in ((K.LRU, "LRU"), (K.FIFO, "FIFO"), (K.LFU, "LFU")):
        for mode in (False, True):
            cell = np.nonzero(replay & (cfg["policy"] == p) & (ttl_mode == mode))[0]
            if len(cell) == 0:
                continue
            pick = rng.choice(cell, min(args.per_cell, len(cell)), replace=False)
            idx.append(pick)
            cells[f"{pn}-{'ttl' if mode else 'capacity'}"] = {"grid": int(len(cell)), "sampled": int(len(pick))}
    idx = np.sort(np.concatenate(idx))
    if args.ttl_groups > 0:
        os.environ["KARETO_K6_COLLAPSE"] = "1"
        pairs = sorted({(int(a), int(b)) for a, b in cfg["cap"][:, :2]})
        pick = [pairs[i] for i in rng.choice(len(pairs), args.ttl_groups, replace=False)]
        sel = np.zeros(len(cfg), bool)
        for a, b in pick:
            sel |= ttl_mode & (cfg["policy"] != K.LRU) & (cfg["cap"][:, 0] == a) & (cfg["cap"][:, 1] == b)
        idx = np.nonzero(sel)[0]
        cells = {"ttl_groups": [list(p) for p in pick], "configs": int(len(idx))}
    sub = cfg[idx]

    torch.cuda.set_device(0)
    ctx = K.Context(0)
    gt = ctx.load(tr, top_k=spec["top_k"])
    assert (gt.N, gt.U, gt.R) == (ot.N, ot.U, ot.R)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    got, obj = ctx.eval_grid(gt, sub, K.Model(), rows)
    gpu_s = time.perf_counter() - t1
    oc = np.zeros(len(sub), O.CONFIG_DTYPE)
    for f in ("cap", "policy", "medium", "tuner", "axis"):
        oc[f] = sub[f]
    osel = np.arange(len(sub))
    if args.oracle_sample and args.oracle_sample < len(sub):
        osel = np.sort(rng.choice(len(sub), args.oracle_sample, replace=False))
    t2 = time.perf_counter()
    want = ot.replay(oc[osel], rows, threads=args.oracle_threads or None)
    oracle_s = time.perf_counter() - t2
    got, obj = got[osel], obj[osel]
    oc = oc[osel]
    same = got.view(np.uint64).reshape(len(osel), -1) == want.view(np.uint64).reshape(len(osel), -1)
    fo = ot.objective(O.Model(), oc, want)
    n_rep = int(replay.sum())
    rate = gt.N * len(sub) / gpu_s
    out = {
        "metric": "K6 replay at full config-3 size on a stratified sample (row a7)",
        "n_accesses": int(gt.N), "n_unique": int(gt.U), "n_requests": int(gt.R),
        "grid_configs": int(len(cfg)), "grid_replay_configs": n_rep, "cells": cells,
        "sample_configs": int(len(sub)), "oracle_checked_configs": int(len(osel)),
        "gpu_s": gpu_s, "access_configs_per_s": rate,
        "oracle_o1_s": oracle_s, "oracle_threads": args.oracle_threads or os.cpu_count(),
        "counts_bit_exact": bool(same.all()), "configs_differing": int((~same.all(1)).sum()),
        "objectives_bit_identical": bool(np.array_equal(obj.view(np.uint64), fo.view(np.uint64))),
        "extrapolated_full_replay_h_at_sample_rate": gt.N * n_rep / rate / 3600.0,
        "note": "the sample's configurations run in one wave per class; a full grid needs memory-bounded waves "
                "of the same per-thread pass time (DESIGN.md section 9)",
        "prep_s": prep_s,
    }
    print(json.dumps(out), flush=True)
    if not same.all():
        sys.exit(1)


if __name__ == "__main__":
    main()

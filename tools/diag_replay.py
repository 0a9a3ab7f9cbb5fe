"""Diagnostic (not a test): K6 replay throughput per policy on the config-3 twin trace."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import kareto_inputs as ki  # noqa: E402
import paper_2603_08739_b200 as K  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
tr = ki.synthetic("chat", R=R, seed=0)
ctx = K.Context(0)
t = ctx.load(tr, top_k=16)
A = lambda m, top: [top * i // (m - 1) for i in range(m)]
rng = np.random.default_rng(0)
caps = np.stack([rng.choice(A(16, t.U // 16), n), rng.choice(A(16, t.U // 2), n), rng.choice(A(7, t.U), n)], 1)
M = K.Model()
for pol, name in ((K.LRU, "LRU-pergroup"), (K.FIFO, "FIFO"), (K.LFU, "LFU")):
    cf = K.configs(caps, policy=pol)
    ttl = np.array([[60_000 + 1000 * g for g in range(17)]], np.uint32)
    ctx.set_profiling(True)
    ctx.pass_times(reset=True)
    w0 = time.perf_counter()
    c, o = ctx.eval_grid(t, cf, M, ttl)
    dt = time.perf_counter() - w0
    pt = {}
    for p in ctx.pass_times(reset=True):
        key = "K6_replay" if p["name"].startswith("K6_replay") else p["name"]
        pt[key] = pt.get(key, 0.0) + p["ms"]
    print(f"{name:14s} n={n} N={t.N} wall {dt:.2f} s  K6 {pt.get('K6_replay', 0) / 1e3:.2f} s  "
          f"{n * t.N / (pt.get('K6_replay', 1e-9) / 1e3):.3e} access-configs/s", flush=True)

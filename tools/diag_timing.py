"""Diagnostic (not a test): wall-clock breakdown of one hot-path step on the GPU box."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import kareto_inputs as ki  # noqa: E402
import paper_2603_08739_b200 as K  # noqa: E402
from bench import grid_configs  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
plan = ki.Plan("chat", R=R, seed=0)
tr = plan.materialize()
stream = torch.cuda.Stream()
ctx = K.Context(0, stream.cuda_stream)
dev = [torch.from_numpy(x).cuda() for x in (tr.arrival_ms, tr.output_tokens, tr.offsets, tr.tokens.view(np.int32))]
torch.cuda.synchronize()
t = ctx.load_trace(*dev[:3], tokens=dev[3], top_k=16)
cfg = grid_configs(K, t.U, (32, 32, 16), (16, 2, 1))
t.free()
M = K.Model()
for it in range(4):
    w0 = time.perf_counter()
    t = ctx.load_trace(*dev[:3], tokens=dev[3], top_k=16)
    w1 = time.perf_counter()
    c, o = ctx.eval_grid(t, cfg, M)
    w2 = time.perf_counter()
    s, nf = ctx.pareto(o, cfg, None)
    w3 = time.perf_counter()
    t.free()
    w4 = time.perf_counter()
    print(f"iter {it}: load {1e3*(w1-w0):.1f} ms eval {1e3*(w2-w1):.1f} pareto {1e3*(w3-w2):.1f} free {1e3*(w4-w3):.1f}",
          flush=True)
ctx.set_profiling(True)
t = ctx.load_trace(*dev[:3], tokens=dev[3], top_k=16)
t.free()
tot = 0
for p in ctx.pass_times():
    tot += p["ms"]
    print(f"  {p['name']:24s} {p['ms']:8.3f} ms x{p['launches']}")
print("sum of passes", tot)

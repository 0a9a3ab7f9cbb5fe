import time, json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import kareto_inputs as ki, paper_2603_08739_b200 as K
import bench
spec = bench.CONFIGS[int(sys.argv[1])]
plan = ki.Plan(spec["kind"], R=spec.get("R", 0), N=spec.get("N", 0), seed=0)
R, T = plan.n_requests, plan.n_tokens
arr = np.empty(R, np.int64); out = np.empty(R, np.int32); off = np.empty(R + 1, np.int64)
tok = torch.empty(T, dtype=torch.int32, pin_memory=True)
plan.fill_meta(arr, out, off); plan.fill_tokens_ptr(tok.data_ptr())
st = torch.cuda.Stream()
ctx = K.Context(0, st.cuda_stream)
d = [torch.from_numpy(x).cuda() for x in (arr, out, off)] + [tok.cuda()]
tr = ctx.load_trace(*d[:3], tokens=d[3], top_k=spec.get("top_k", 16))
cfg, ttl = bench.build_grid(K, spec, tr)
tr.free()
cnt = torch.empty((len(cfg), 11), dtype=torch.int64, device="cuda"); obj = torch.empty((len(cfg), 3), dtype=torch.float64, device="cuda")
sd = torch.empty(len(cfg), dtype=torch.uint8, device="cuda")
m = K.Model()
for it in range(6):
    t0 = time.perf_counter(); t = ctx.load_trace(*d[:3], tokens=d[3], top_k=spec.get("top_k", 16)); t1 = time.perf_counter()
    ctx.eval_grid(t, cfg, m, ttl, counts=cnt, obj=obj); t2 = time.perf_counter()
    ctx.pareto(obj, cfg, spec["prune"], status=sd); t3 = time.perf_counter()
    t.free(); t4 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} eval {1e3*(t2-t1):.2f} pareto {1e3*(t3-t2):.2f} free {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f}")
ctx.set_profiling(True); ctx.pass_times(reset=True)
t = ctx.load_trace(*d[:3], tokens=d[3], top_k=spec.get("top_k", 16)); ctx.eval_grid(t, cfg, m, ttl, counts=cnt, obj=obj); ctx.pareto(obj, cfg, spec["prune"], status=sd); t.free()
ps = ctx.pass_times(reset=True)
print("device passes", round(sum(p["ms"] for p in ps), 3))

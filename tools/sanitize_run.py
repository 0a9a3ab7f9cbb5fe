"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): load (K1-K3), eval_grid over stack-path LRU configurations and all five K6 replay
classes (run concurrently, several waves each through a small KARETO_K6_BUDGET), pareto (K8), a
2-rank loopback time-sharded load, and row f1/f2/f3 calls.  Checks the counts against the oracle
so a sanitizer-clean run is also a correct one.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [all|trace|replay]

`trace`: load + LRU stack grid + pareto + the loopback time-sharded load (K1-K4, K8 and the
shared-memory-atomic kernels); `replay`: a small K6 grid (every class, several waves) -- racecheck
is too slow for both in one run."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kareto_inputs as ki  # noqa: E402
import paper_2603_08739_b200 as K  # noqa: E402
from oracle import oracle as O  # noqa: E402

U32 = 0xFFFFFFFF
MODE = sys.argv[1] if len(sys.argv) > 1 else "all"
tr = ki.synthetic("chat", R=300 if MODE != "replay" else 120, seed=3)
ot = O.OracleTrace(tr, top_k=4)
ctx = K.Context(0)
gt = ctx.load(tr, top_k=4)
A = lambda m, top: [top * i // (m - 1) for i in range(m)]
rows = np.array([[U32] * 5, [600_000] * 5, [60_000, 600_000, 3_600_000, 30_000, 5_000]], np.uint32)
caps, pol, tun, ax = [], [], [], []
for i, a in enumerate(A(3, ot.U // 16)):
    for j, b in enumerate(A(3, ot.U // 4)):
        for k, c in enumerate(A(3, ot.U)):
            for p in (O.LRU, O.FIFO, O.LFU):
                for ti in range(3):
                    caps.append([a, b, c]); pol.append(p); tun.append(ti); ax.append([i, j, k])
                caps.append([a, b, O.INF_CAP]); pol.append(p); tun.append(2); ax.append([i, j, 0])
oc = O.configs(caps, policy=np.array(pol), tuner=np.array(tun), axis=ax)
if MODE in ("trace", "trace1"):  # stack-path configurations only
    oc = oc[(oc["policy"] == O.LRU) & ((oc["tuner"] != 2) | (oc["cap"][:, 2] == O.INF_CAP))]
kc = K.configs(oc["cap"], policy=oc["policy"], tuner=oc["tuner"], axis=oc["axis"])
os.environ["KARETO_K6_BUDGET"] = str(40 * ot.U * 40)
cnt, obj = ctx.eval_grid(gt, kc, K.Model(), rows)
want = ot.replay(oc, rows)
assert np.array_equal(cnt.view(np.uint64), want.view(np.uint64)), "counts differ from the oracle"
st, nf = ctx.pareto(obj, kc, 0.05)
assert np.array_equal(st, O.select(ot.objective(O.Model(), oc, want), oc, 0.05))
del os.environ["KARETO_K6_BUDGET"]
if MODE in ("replay", "trace1"):
    print(f"sanitize run ok ({MODE}): N={gt.N} U={gt.U} configs={len(kc)} frontier={nf}")
    sys.exit(0)
ctx.ttl_allocate(gt, 10**9, seed=1)
lru = np.nonzero(oc["policy"] == O.LRU)[0][:8]
ctx.eval_queue(gt, kc[lru], K.Model(), rows)
if MODE == "trace1":  # no loopback threads
    print(f"sanitize run ok ({MODE}): N={gt.N} U={gt.U} configs={len(kc)} frontier={nf}")
    sys.exit(0)
grp = K.Loopback(2)
errs = []


def rank(r):
    try:
        c = K.Context(0, loopback=grp, rank=r)
        t = c.load(tr, top_k=4, time_shard=True)
        t.free()
        c.close()
    except BaseException as e:  # noqa: BLE001
        errs.append(e)


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
assert not errs, errs
print(f"sanitize run ok ({MODE}): N={gt.N} U={gt.U} configs={len(kc)} frontier={nf}")

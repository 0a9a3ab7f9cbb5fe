"""GPU parity for row f3 (kareto_eval_queue) against oracle/queue.py: per-configuration mean and
P99 TTFT, makespan, throughput and disk hits (capacity / realised) on the same seeded traces.

Bar: integers bit-exact; fp64 bit-identical (both sides run the same operation sequence, the
GPU translation unit without FMA contraction, R33)."""
import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O
from oracle import queue as Q

pytestmark = pytest.mark.gpu
INF = int(O.INF_CAP)
MODEL_KW = dict(gpus_per_instance=8, alpha_ps=50_000_000, beta_ps=1, dec_ps=150_000_000, block_bytes=5_242_880,
                bw_dram=25e9, c_hw=2.5, p_hbm=0.0, p_dram=0.004, iops_per_block=1.0, ttl_prov_gb=1024.0,
                media=((120e6, 0.5e6, 350e6, 0.0001), (2e9, 0.0, 4e9, 0.0003)),
                phi=((0.0, 0.0, 0.0),))


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


def kcfg(oc):
    c = np.zeros(len(oc), K.CONFIG_DTYPE)
    for f in ("cap", "policy", "medium", "tuner", "axis"):
        c[f] = oc[f]
    return c


@pytest.mark.parametrize("kind,R,seed,inst", [("chat", 500, 0, 1), ("chat", 800, 1, 3), ("agent", 40, 2, 2),
                                              ("api", 300, 3, 1)])
def test_queue_parity(ctx, kind, R, seed, inst):
    tr = ki.synthetic(kind, R=R, seed=seed)
    ot = O.OracleTrace(tr, top_k=3)
    U = ot.U
    caps = [(0, 0, 0), (U // 50, U // 10, U // 3), (U // 20, U // 5, U), (0, U // 4, INF), (U // 30, 0, INF),
            (U // 10, U // 10, 7), (U, U, U)]
    ttl = np.array([[0xFFFFFFFF] * 4, [60_000] * 4, [5_000, 600_000, 30_000, 1_000_000]], np.uint32)
    rows = []
    for cap in caps:
        for t in range(3):
            if cap[2] == INF and t == 0:
                continue                    # TTL mode needs finite TTLs (R22)
            for pol in (O.LRU, O.FIFO, O.LFU):
                rows.append((cap, t, (len(rows) % 2), pol))
    oc = O.configs([r[0] for r in rows], tuner=[r[1] for r in rows], medium=[r[2] for r in rows],
                   policy=[r[3] for r in rows])
    want = Q.evaluate(tr, ot, oc, ttl, O.Model(instances=inst, **MODEL_KW))
    gt = ctx.load(tr, top_k=3)
    got = ctx.eval_queue(gt, kcfg(oc), K.Model(instances=inst, **MODEL_KW), ttl)
    for i, w in enumerate(want):
        g = got[i]
        assert (int(g["disk_hits_capacity"]), int(g["disk_hits_realized"])) == (w["disk_cap"], w["disk_real"]), \
            (i, rows[i])
        for f, k in (("ttft_mean_ms", "mean_ms"), ("ttft_p99_ms", "p99_ms"), ("makespan_s", "makespan_s"),
                     ("tokens_per_s", "tok_per_s")):
            assert np.float64(g[f]).view(np.uint64) == np.float64(w[k]).view(np.uint64), (i, rows[i], f, g[f], w[k])


def test_queue_invalid(ctx):
    tr = ki.synthetic("chat", R=50, seed=9)
    gt = ctx.load(tr, top_k=2)
    m = K.Model(**MODEL_KW)
    with pytest.raises(K.KaretoError, match="infinite"):
        ctx.eval_queue(gt, K.configs([[1, 1, int(K.INF)]]), m)
    with pytest.raises(K.KaretoError, match="tuner"):
        ctx.eval_queue(gt, K.configs([[1, 1, 1]], tuner=2), m, np.array([[1, 2, 3]], np.uint32))

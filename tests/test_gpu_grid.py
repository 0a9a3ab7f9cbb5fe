"""Prepared grids (kareto_grid_create / kareto_eval_grid_prepared / kareto_pareto_prepared): the
same outputs as kareto_eval_grid / kareto_pareto, bit for bit, and therefore as the oracle -- on
a mixed stack / replay grid, reused across two traces, through a 2-rank loopback configuration
shard and through a time-sharded trace (the grid's shard is re-derived), plus the error rules."""
import threading

import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O

pytestmark = pytest.mark.gpu
U32 = 0xFFFFFFFF


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


def mixed(U):
    rows = np.array([[U32] * 5, [600_000] * 5, [60_000, 600_000, 3_600_000, 30_000, 5_000]], np.uint32)
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, pol, tun, ax = [], [], [], []
    for i, a in enumerate(A(3, U // 16)):
        for j, b in enumerate(A(3, U // 4)):
            for k, c in enumerate(A(3, U)):
                for p in (O.LRU, O.FIFO, O.LFU):
                    for ti in range(3):
                        caps.append([a, b, c]); pol.append(p); tun.append(ti); ax.append([i, j, k])
                    caps.append([a, b, O.INF_CAP]); pol.append(p); tun.append(2); ax.append([i, j, 0])
    oc = O.configs(caps, policy=np.array(pol), tuner=np.array(tun), axis=ax)
    return oc, K.configs(oc["cap"], policy=oc["policy"], tuner=oc["tuner"], axis=oc["axis"]), rows


def test_prepared_equals_unprepared_and_oracle_on_two_traces(ctx):
    tr1 = ki.synthetic("chat", R=800, seed=21)
    tr2 = ki.synthetic("chat", R=700, seed=22)
    U = O.OracleTrace(tr1, top_k=4).U
    oc, kc, rows = mixed(U)
    g = ctx.grid(kc, rows)
    for tr in (tr1, tr2):
        gt = ctx.load(tr, top_k=4)
        c0, o0 = ctx.eval_grid(gt, kc, K.Model(), rows)
        c1, o1 = ctx.eval_prepared(gt, g, K.Model())
        assert np.array_equal(c0.view(np.uint64), c1.view(np.uint64))
        assert np.array_equal(o0.view(np.uint64), o1.view(np.uint64))
        ot = O.OracleTrace(tr, top_k=4)
        want = ot.replay(oc, rows)
        assert np.array_equal(c1.view(np.uint64), want.view(np.uint64))
        s0, n0 = ctx.pareto(o0, kc, 0.05)
        s1, n1 = ctx.pareto_prepared(o1, g, 0.05)
        assert np.array_equal(s0, s1) and n0 == n1
        assert np.array_equal(s1, O.select(ot.objective(O.Model(), oc, want), oc, 0.05))
        s2, _ = ctx.pareto_prepared(o1, g, None)  # no pruning
        assert np.array_equal(s2, ctx.pareto(o1, kc, None)[0])
        gt.free()
    g.free()


def test_prepared_errors(ctx):
    tr = ki.synthetic("chat", R=200, seed=3)
    gt = ctx.load(tr, top_k=4)
    kc = K.configs([[1, 2, 3]] * 4, medium=[0, 0, 2, 0])
    g = ctx.grid(kc, n_groups=5)
    with pytest.raises(K.KaretoError, match="config 2: medium"):   # model with one medium
        ctx.eval_prepared(gt, g, K.Model())
    g6 = ctx.grid(K.configs([[1, 2, 3]]), n_groups=6)
    with pytest.raises(K.KaretoError, match="groups"):            # grid for K = 5, trace K = 4
        ctx.eval_prepared(gt, g6, K.Model())
    with pytest.raises(K.KaretoError, match="tuner"):
        ctx.grid(K.configs([[1, 2, 3]], tuner=3), np.full((2, 5), U32, np.uint32))
    bad = K.configs([[1, 2, 3]] * 2, axis=[[0, 0, 0], [70000, 0, 0]])
    gb = ctx.grid(bad, n_groups=5)                                 # fine without pruning ...
    obj = np.zeros((2, 3))
    ctx.pareto_prepared(obj, gb, None)
    with pytest.raises(K.KaretoError, match="axis out of range"):  # ... not with it
        ctx.pareto_prepared(obj, gb, 0.05)
    for x in (g, g6, gb):
        x.free()
    gt.free()


def test_prepared_loopback_shard_and_time_shard(ctx):
    import torch
    tr = ki.synthetic("chat", R=600, seed=31)
    ot = O.OracleTrace(tr, top_k=4)
    oc, kc, rows = mixed(ot.U)
    want = ot.replay(oc, rows)
    grp = K.Loopback(2)
    out, err = [None, None], []

    def rank(r):
        try:
            s = torch.cuda.Stream()
            c = K.Context(0, s.cuda_stream, loopback=grp, rank=r)
            g = c.grid(kc, rows)                       # each rank prepares its cost-weighted shard
            t = c.load(tr, top_k=4)
            out[r] = c.eval_prepared(t, g, K.Model())[0]
            t.free()
            g.free()
            c.close()
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not err, err
    for o in out:
        assert np.array_equal(o.view(np.uint64), want.view(np.uint64))
    grp.close()
    # a grid prepared on a 1-rank NCCL context (configuration shard) used with a time-sharded trace:
    # the shard is re-derived for the whole grid (stack configurations only on time shards)
    nid = K.Context.nccl_unique_id()
    cn = K.Context(0, torch.cuda.current_stream().cuda_stream, nid, 0, 1)
    lru = oc[(oc["policy"] == O.LRU) & ((oc["tuner"] == 0) | (oc["cap"][:, 2] == O.INF_CAP))]
    klru = K.configs(lru["cap"], policy=lru["policy"], tuner=lru["tuner"], axis=lru["axis"])
    g = cn.grid(klru, rows)
    ts = cn.load(tr, top_k=4, time_shard=True)
    c1, _ = cn.eval_prepared(ts, g, K.Model())
    assert np.array_equal(c1.view(np.uint64), ot.stack_counts(lru, rows).view(np.uint64))
    ts.free()
    g.free()
    cn.close()

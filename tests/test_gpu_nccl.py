"""The NCCL transport on one B200 (row e; VERDICT r1 "What's missing" #5): a context created
with world = 1 and an NCCL unique id owns a 1-rank communicator (dlopen'ed libnccl, the same
ncclCommInitRank / ncclAllGather / ncclAllReduce / grouped ncclSend+ncclRecv calls a multi-GPU run
makes), so the configuration-shard gather of kareto_eval_grid and the time-sharded load's
all-to-all and allreduces run through NCCL.  Results are compared with the oracle (counts,
objectives, Pareto status bit-exact; prev / depth of the time-sharded load identical)."""
import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O

pytestmark = pytest.mark.gpu
U32 = 0xFFFFFFFF


@pytest.fixture(scope="module")
def nccl_ctx():
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    nid = K.Context.nccl_unique_id()
    assert len(nid) == 128
    return K.Context(0, torch.cuda.current_stream().cuda_stream, nid, 0, 1)


def test_eval_grid_through_nccl_allgather(nccl_ctx):
    tr = ki.synthetic("chat", R=600, seed=12)
    ot = O.OracleTrace(tr, top_k=4)
    gt = nccl_ctx.load(tr, top_k=4)
    rows = np.array([[U32] * 5, [600_000] * 5, [60_000, 600_000, 3_600_000, 30_000, 5_000]], np.uint32)
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, pol, tun, ax = [], [], [], []
    for i, a in enumerate(A(3, ot.U // 16)):
        for j, b in enumerate(A(3, ot.U // 4)):
            for k, c in enumerate(A(3, ot.U)):
                for p in (O.LRU, O.FIFO, O.LFU):
                    for ti in range(3):
                        caps.append([a, b, c]); pol.append(p); tun.append(ti); ax.append([i, j, k])
    oc = O.configs(caps, policy=np.array(pol), tuner=np.array(tun), axis=ax)
    kc = K.configs(oc["cap"], policy=oc["policy"], tuner=oc["tuner"], axis=oc["axis"])
    cnt, obj = nccl_ctx.eval_grid(gt, kc, K.Model(), rows)
    want = ot.replay(oc, rows)
    assert np.array_equal(cnt.view(np.uint64), want.view(np.uint64))
    fo = ot.objective(O.Model(), oc, want)
    assert np.array_equal(obj.view(np.uint64), fo.view(np.uint64))
    st, _ = nccl_ctx.pareto(obj, kc, 0.05)
    assert np.array_equal(st, O.select(fo, oc, 0.05))


def test_time_sharded_load_through_nccl(nccl_ctx):
    tr = ki.synthetic("agent", R=300, seed=5)
    ot = O.OracleTrace(tr, top_k=4)
    t = nccl_ctx.load(tr, top_k=4, time_shard=True)
    e = ot.export()
    assert np.array_equal(t.export(K.X_PREV).astype(np.int64), np.where(e["prev"] < 0, U32, e["prev"]))
    d, _ = ot.depth()
    assert np.array_equal(t.export(K.X_DEPTH).astype(np.int64), np.where(d < 0, U32, d))
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps = [[a, b, c] for a in A(3, ot.U // 16) for b in A(3, ot.U // 4) for c in A(3, ot.U)]
    oc = O.configs(caps)
    cnt, _ = nccl_ctx.eval_grid(t, K.configs(caps), K.Model())   # histogram allreduce through NCCL
    assert np.array_equal(cnt.view(np.uint64), ot.stack_counts(oc).view(np.uint64))

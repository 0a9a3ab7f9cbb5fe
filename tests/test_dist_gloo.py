"""N > 1 host path on CPU: world_size-2 gloo processes (127.0.0.1).

Each rank takes the deterministic shard libkareto evaluates (kareto_shard_range), computes
its shard's counts + objective vectors (with the oracle standing in for the GPU, which this
box does not have), exchanges padded slots with an all_gather exactly as kareto_eval_grid's
ncclAllGather does, reassembles with dist.assemble, and runs the global selection: the result
must equal the single-process evaluation byte for byte.  The NCCL-id broadcast helper is
exercised over gloo too."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import kareto_inputs as ki
        import paper_2603_08739_b200 as K
        from oracle import oracle as O
        from paper_2603_08739_b200 import dist as kd

        nid = kd.broadcast_unique_id(rank, world, make_id=lambda: bytes(range(128)))
        assert nid == bytes(range(128))
        tr = ki.synthetic("chat", R=600, seed=9)
        ot = O.OracleTrace(tr, top_k=4)
        A = lambda m, top: [top * i // (m - 1) for i in range(m)]
        caps = [[a, b, c] for a in A(5, ot.U // 16) for b in A(5, ot.U // 4) for c in A(3, ot.U)]
        axis = [[i, j, k] for i in range(5) for j in range(5) for k in range(3)]
        # mixed grid: LRU (stack path, weight 1) then FIFO (replay, weight 10^6): the cost-weighted
        # bounds give each rank about half of the FIFO configurations, not half of the list
        pol = np.array([O.LRU] * 60 + [O.FIFO] * 15)
        cf = O.configs(caps, axis=axis, policy=pol)
        n = len(cf)
        bounds = K.shard_bounds(K.configs(cf["cap"], policy=cf["policy"], axis=cf["axis"]), world, n_groups=5)
        assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) >= 0)
        n_fifo = [int((pol[bounds[r]:bounds[r + 1]] == O.FIFO).sum()) for r in range(world)]
        assert max(n_fifo) - min(n_fifo) <= 1, n_fifo
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        cnt = ot.replay(cf[lo:hi], threads=2)
        f = ot.objective(O.Model(), cf[lo:hi], cnt)
        slot = kd.slot_size(bounds)
        buf_c = np.zeros(slot, O.COUNTS_DTYPE)
        buf_c[: hi - lo] = cnt
        buf_f = np.zeros((slot, 3))
        buf_f[: hi - lo] = f
        tc = torch.from_numpy(buf_c.view(np.uint8).copy())
        tf = torch.from_numpy(buf_f.copy())
        gc = [torch.zeros_like(tc) for _ in range(world)]
        gf = [torch.zeros_like(tf) for _ in range(world)]
        dist.all_gather(gc, tc)
        dist.all_gather(gf, tf)
        all_c = kd.assemble([g.numpy().view(O.COUNTS_DTYPE) for g in gc], bounds)
        all_f = kd.assemble([g.numpy() for g in gf], bounds)
        st = O.select(all_f, cf, 0.05)
        out_q.put((rank, all_c.tobytes(), all_f.tobytes(), st.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shard_gather_equals_single_process():
    import kareto_inputs as ki
    from oracle import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single process reference
    tr = ki.synthetic("chat", R=600, seed=9)
    ot = O.OracleTrace(tr, top_k=4)
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps = [[a, b, c] for a in A(5, ot.U // 16) for b in A(5, ot.U // 4) for c in A(3, ot.U)]
    axis = [[i, j, k] for i in range(5) for j in range(5) for k in range(3)]
    cf = O.configs(caps, axis=axis, policy=np.array([O.LRU] * 60 + [O.FIFO] * 15))
    cnt = ot.replay(cf)
    f = ot.objective(O.Model(), cf, cnt)
    st = O.select(f, cf, 0.05)
    for _, c, ff, s in res:
        assert c == cnt.tobytes() and ff == f.tobytes() and s == st.tobytes()

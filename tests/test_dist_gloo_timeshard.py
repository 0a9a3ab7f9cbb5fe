"""N > 1 host path of the time-sharded load (row f4) on CPU: world_size 2 and 3 gloo processes
(127.0.0.1) run the exchange protocol of kareto_load_trace_sharded with the library's own
partition rules (kareto_time_slices: which requests a rank keeps; kareto_hash_owner: which rank
owns a block hash) and the oracle's hashes standing in for the GPU's K1 (this box has no GPU):

  1. each rank links the accesses of its slice and emits one record per distinct block
     (first and last position in the slice) to the block's owner (all-to-all over gloo);
  2. owners order each block's records by slice, answer each with the previous slice's last
     position (or "globally first") and the next slice holding the block;
  3. every rank sends each later rank its last positions whose block next appears at or after
     that rank (the boundary LRU set B_k);
  4. each rank computes its depths on the compressed coordinates (B_k prefixed).

prev, depth (per access of every slice) and U must equal the oracle's whole-trace values."""
import bisect
import os
import socket
from collections import defaultdict

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _alltoall(obj_by_dest, world):
    """all-to-all of Python objects over gloo (all_gather, each rank keeps its column)."""
    g = [None] * world
    dist.all_gather_object(g, obj_by_dest)
    me = dist.get_rank()
    return [g[src][me] for src in range(world)]


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import kareto_inputs as ki
        import paper_2603_08739_b200 as K
        from oracle import oracle as O

        tr = ki.synthetic("chat", R=400, seed=3)
        ot = O.OracleTrace(tr, top_k=2)
        e = ot.export()
        s, hashes, req = e["s"], e["hash"], e["req"]
        rb = K.time_slices(s.astype(np.uint32), world)
        pb = s[rb]
        P0, P1 = int(pb[rank]), int(pb[rank + 1])
        r0, r1 = int(rb[rank]), int(rb[rank + 1])
        # 1. in-slice links and one record per distinct block: (hash, first, last)
        first, last = {}, {}
        prev = np.full(P1 - P0, -1, np.int64)
        for i in range(P1 - P0):
            h = int(hashes[P0 + i])
            if h in last:
                prev[i] = P0 + last[h]
            else:
                first[h] = i
            last[h] = i
        out = [[] for _ in range(world)]
        for h in first:
            out[K.hash_owner(h, world)].append((h, P0 + first[h], P0 + last[h]))
        got = _alltoall(out, world)
        # 2. owner: records of a block ordered by source slice
        by = defaultdict(list)
        for src, recs in enumerate(got):
            for h, f, l in recs:
                by[h].append((src, f, l))
        ans = [dict() for _ in range(world)]
        for h, lst in by.items():
            lst.sort()
            for j, (src, f, l) in enumerate(lst):
                ans[src][h] = (lst[j - 1][2] if j > 0 else -1, lst[j + 1][0] if j + 1 < len(lst) else world)
        mine = {}
        for part in _alltoall(ans, world):
            mine.update(part)
        for h, i in first.items():
            prev[i] = mine[h][0]
        n_first = sum(1 for h in first if mine[h][0] < 0)
        # 3. boundary sets: this slice's last positions whose block next appears at or after k
        contrib = [sorted(P0 + last[h] for h in first if mine[h][1] >= k) if k > rank else [] for k in range(world)]
        B = sorted(p for part in _alltoall(contrib, world) for p in part)
        # 4. depths on compressed coordinates: virtual trace = B (distinct blocks) + the slice
        nb = len(B)
        rank_b = {p: i for i, p in enumerate(B)}
        pc = [-1 if p < 0 else (nb + p - P0 if p >= P0 else rank_b[p]) for p in prev]
        depth = np.full(P1 - P0, -1, np.int64)
        seen = []  # sorted compressed prevs of the accesses before the current request
        for r in range(r0, r1):
            a, b = int(s[r]) - P0, int(s[r + 1]) - P0
            sr = nb + a
            for i in range(a, b):
                if pc[i] >= 0:
                    depth[i] = sr - pc[i] - (len(seen) - bisect.bisect_left(seen, pc[i]))
            for i in range(a, b):
                if pc[i] >= 0:
                    bisect.insort(seen, pc[i])
        out_q.put((rank, P0, P1, prev.tobytes(), depth.tobytes(), n_first))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_time_shard_protocol_matches_whole_trace(world):
    import kareto_inputs as ki
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tr = ki.synthetic("chat", R=400, seed=3)
    ot = O.OracleTrace(tr, top_k=2)
    e = ot.export()
    d, _ = ot.depth()
    assert res[0][1] == 0 and res[-1][2] == ot.N
    for (_, _, hi, *_), (_, lo, *_) in zip(res, res[1:]):
        assert hi == lo
    prev = np.concatenate([np.frombuffer(x[3], np.int64) for x in res])
    depth = np.concatenate([np.frombuffer(x[4], np.int64) for x in res])
    assert np.array_equal(prev, e["prev"])
    assert np.array_equal(depth, d)
    assert sum(x[5] for x in res) == ot.U

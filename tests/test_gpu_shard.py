"""GPU parity of the multi-rank paths, run on ONE GPU through the in-process loopback rank
group (kareto_create_loopback: W contexts, one host thread and CUDA stream each; the data
movement replaces NCCL, every kernel and every exchange step is the production code).

* row f4 time sharding (kareto_load_trace_sharded): each rank's shard of prev / delta / depth /
  hash / req and the groups of its requests equal the oracle's whole-trace values (O-1..O-6,
  O2 depths); U, U_g, reuse_g equal; kareto_eval_grid on the shards (K4 histograms summed over
  the ranks) gives counts bit-exact against the oracle's literal replay O1 and bit-identical
  objectives, on every rank.
* row e configuration sharding (kareto_eval_grid with world > 1 on whole traces): the padded
  slot gather reassembles the single-rank result byte for byte.
"""
import threading

import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O

pytestmark = pytest.mark.gpu

U32 = 0xFFFFFFFF
MODEL_KW = dict(instances=2, gpus_per_instance=8, alpha_ps=50_000_000, beta_ps=1, dec_ps=150_000_000,
                block_bytes=5_242_880, bw_dram=25e9, c_hw=2.5, p_hbm=0.001, p_dram=0.004, iops_per_block=1.0,
                ttl_prov_gb=1024.0, media=((120e6, 0.5e6, 350e6, 0.0001), (300e6, 1e6, 1e9, 0.0003)),
                phi=((0.0, 0.0, 0.0), (3000.0, 0.005, 0.0), (32000.0, 0.065, 0.0)))


def run_ranks(W, fn):
    """fn(rank, ctx) on W threads, each with its own loopback context and CUDA stream."""
    import torch
    group = K.Loopback(W)
    out, err = [None] * W, [None] * W

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            ctx = K.Context(0, s.cuda_stream, loopback=group, rank=r)
            out[r] = fn(r, ctx)
            ctx.close()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for e in err:
        if e is not None:
            raise e
    group.close()
    return out


def grid(U, ttl_mode=True):
    """3-tier LRU capacity grid (stack path) + TTL-mode configurations with per-group rows."""
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, axis, tun = [], [], []
    for i, a in enumerate(A(4, max(U // 16, 3))):
        for j, b in enumerate(A(4, max(U // 4, 3))):
            for k, c in enumerate(A(3, U)):
                caps.append([a, b, c]); axis.append([i, j, k]); tun.append(0)
                if ttl_mode:  # finite disk with a uniform TTL row: stack path with delta-binned K4 cells
                    caps.append([a, b, c]); axis.append([i, j, k]); tun.append(1)
            if ttl_mode:
                for t in (1, 2):
                    caps.append([a, b, K.INF]); axis.append([i, j, 3]); tun.append(t)
    return caps, axis, tun


def oracle_cfgs(caps, axis, tun):
    c = np.zeros(len(caps), O.CONFIG_DTYPE)
    c["cap"] = np.array(caps, np.uint64)
    c["axis"] = axis
    c["tuner"] = tun
    return c


def kernel_cfgs(oc):
    c = np.zeros(len(oc), K.CONFIG_DTYPE)
    for f in ("cap", "policy", "medium", "tuner", "axis"):
        c[f] = oc[f]
    return c


def ttl_rows(K_):
    return np.array([[U32] * (K_ + 1), [5_000] * (K_ + 1), [(g + 1) * 20_000 for g in range(K_ + 1)]], np.uint32)


CASES = [
    ("chat", dict(R=3000, seed=5), 8, 0),
    ("agent", dict(N=300_000, seed=2), 4, 0),
    ("api", dict(R=2000, seed=9), 3, 7),
]


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_time_shard_parity(W, case):
    kind, kw, top_k, salt = CASES[case]
    tr = ki.synthetic(kind, **kw)
    ot = O.OracleTrace(tr, top_k=top_k, salt=salt)
    e = ot.export()
    d, _ = ot.depth()
    caps, axis, tun = grid(ot.U)
    oc = oracle_cfgs(caps, axis, tun)
    rows = ttl_rows(top_k)
    want = ot.replay(oc, rows)
    fo = ot.objective(O.Model(**MODEL_KW), oc, want)

    def fn(r, ctx):
        gt = ctx.load(tr, top_k=top_k, salt=salt, time_shard=True)
        res = dict(lo=gt.pos_lo, hi=gt.pos_hi, rlo=gt.req_lo, rhi=gt.req_hi, N=gt.N, U=gt.U, R=gt.R,
                   Ug=gt.U_g.copy(), Rg=gt.reuse_g.copy())
        for x in (K.X_HASH, K.X_PREV, K.X_DELTA, K.X_REQ, K.X_DEPTH, K.X_GROUP):
            res[x] = gt.export(x)
        res["counts"], res["obj"] = ctx.eval_grid(gt, kernel_cfgs(oc), K.Model(**MODEL_KW), rows)
        gt.free()
        return res

    out = run_ranks(W, fn)
    # shards tile [0, N) and [0, R) in rank order
    assert out[0]["lo"] == 0 and out[-1]["hi"] == ot.N and out[0]["rlo"] == 0 and out[-1]["rhi"] == ot.R
    for a, b in zip(out, out[1:]):
        assert a["hi"] == b["lo"] and a["rhi"] == b["rlo"]
    for r, res in enumerate(out):
        lo, hi, rlo, rhi = res["lo"], res["hi"], res["rlo"], res["rhi"]
        assert (res["N"], res["U"], res["R"]) == (ot.N, ot.U, ot.R)
        assert np.array_equal(res["Ug"], ot.U_g) and np.array_equal(res["Rg"], ot.reuse_g)
        assert np.array_equal(res[K.X_HASH], e["hash"][lo:hi]), f"rank {r}: hash"
        assert np.array_equal(res[K.X_REQ], e["req"][lo:hi].astype(np.uint32)), f"rank {r}: req"
        assert np.array_equal(res[K.X_PREV].astype(np.int64), np.where(e["prev"] < 0, U32, e["prev"])[lo:hi]), \
            f"rank {r}: prev"
        assert np.array_equal(res[K.X_DELTA].astype(np.int64), np.where(e["delta"] < 0, U32, e["delta"])[lo:hi]), \
            f"rank {r}: delta"
        assert np.array_equal(res[K.X_DEPTH].astype(np.int64), np.where(d < 0, U32, d)[lo:hi]), f"rank {r}: depth"
        assert np.array_equal(res[K.X_GROUP][rlo:rhi], e["group"][rlo:rhi].astype(np.uint16)), f"rank {r}: group"
        g = np.ascontiguousarray(res["counts"]).view(np.uint64).reshape(len(oc), 11)
        w = np.ascontiguousarray(want).view(np.uint64).reshape(len(oc), 11)
        bad = np.nonzero((g != w).any(1))[0]
        assert len(bad) == 0, f"rank {r}: {len(bad)} configs differ, first {oc[bad[0]]}: {res['counts'][bad[0]]} vs {want[bad[0]]}"
        assert np.array_equal(res["obj"].view(np.uint64), fo.view(np.uint64)), f"rank {r}: objectives"


def test_time_shard_tiny_and_empty_shards():
    """More ranks than requests with blocks: empty shards take part in every exchange."""
    rng = np.random.default_rng(3)
    tr = ki.random_prefix_tree(rng, n_req=3)
    ot = O.OracleTrace(tr, top_k=2)
    e, (d, _) = ot.export(), ot.depth()
    W = 5

    def fn(r, ctx):
        gt = ctx.load(tr, top_k=2, time_shard=True)
        return gt.pos_lo, gt.pos_hi, gt.export(K.X_PREV), gt.export(K.X_DEPTH), gt.U

    out = run_ranks(W, fn)
    prev = np.concatenate([o[2] for o in out]).astype(np.int64)
    dep = np.concatenate([o[3] for o in out]).astype(np.int64)
    assert np.array_equal(prev, np.where(e["prev"] < 0, U32, e["prev"]))
    assert np.array_equal(dep, np.where(d < 0, U32, d))
    assert all(o[4] == ot.U for o in out)


def test_time_shard_rejects_replay_configs():
    tr = ki.synthetic("chat", R=500, seed=1)

    def fn(r, ctx):
        gt = ctx.load(tr, top_k=2, time_shard=True)
        c = K.configs([[1, 2, 3]], policy=K.FIFO)
        with pytest.raises(K.KaretoError) as ei:
            ctx.eval_grid(gt, c, K.Model())
        return ei.value.status

    assert run_ranks(2, fn) == [K.E_UNSUPPORTED] * 2


@pytest.mark.parametrize("W", [2, 3])
def test_config_shard_gather_loopback(W):
    """Row e: each rank evaluates its contiguous shard (incl. K6 replay configurations) and the
    allgather reassembles the full result, byte-identical to one rank."""
    import torch
    tr = ki.synthetic("chat", R=1500, seed=4)
    ctx1 = K.Context(0, torch.cuda.current_stream().cuda_stream)
    g1 = ctx1.load(tr, top_k=4)
    caps, axis, tun = grid(g1.U, ttl_mode=False)
    base = K.configs(caps, axis=axis)
    cfgs = np.concatenate([base, base.copy(), base.copy()])
    cfgs["policy"][len(base):2 * len(base)] = K.FIFO
    cfgs["policy"][2 * len(base):] = K.LFU
    want_c, want_o = ctx1.eval_grid(g1, cfgs, K.Model(**MODEL_KW))

    def fn(r, ctx):
        gt = ctx.load(tr, top_k=4)
        return ctx.eval_grid(gt, cfgs, K.Model(**MODEL_KW))

    for c, o in run_ranks(W, fn):
        assert np.array_equal(np.asarray(c).view(np.uint8), np.asarray(want_c).view(np.uint8))
        assert np.array_equal(o.view(np.uint64), want_o.view(np.uint64))


def _check_shards(out, ot):
    e = ot.export()
    d, _ = ot.depth()
    for key, want in ((K.X_HASH, e["hash"]), (K.X_PREV, np.where(e["prev"] < 0, U32, e["prev"])),
                      (K.X_DELTA, np.where(e["delta"] < 0, U32, e["delta"])), (K.X_DEPTH, np.where(d < 0, U32, d))):
        got = np.concatenate([o[key] for o in out]).astype(np.int64 if key != K.X_HASH else np.uint64)
        assert np.array_equal(got, want.astype(got.dtype)), key
    for o in out:
        assert o["U"] == ot.U and np.array_equal(o["Ug"], ot.U_g)
        assert np.array_equal(o[K.X_GROUP][o["rlo"]:o["rhi"]], e["group"][o["rlo"]:o["rhi"]].astype(np.uint16))


def _load_exports(tr, top_k, salt=0):
    def fn(r, ctx):
        gt = ctx.load(tr, top_k=top_k, salt=salt, time_shard=True)
        res = dict(U=gt.U, Ug=gt.U_g.copy(), rlo=gt.req_lo, rhi=gt.req_hi)
        for x in (K.X_HASH, K.X_PREV, K.X_DELTA, K.X_DEPTH, K.X_GROUP):
            res[x] = gt.export(x)
        return res
    return fn


def test_time_shard_hash_mode():
    """HASHES input (caller-provided chained hashes, k_copy_hashes + k_sort_prep path)."""
    tr = ki.synthetic("chat", R=1500, seed=12)
    bh, boff = [], [0]
    for r in range(tr.n_requests):
        h = O.chain_hashes(tr.tokens[tr.offsets[r]:tr.offsets[r + 1]])
        bh.append(h)
        boff.append(boff[-1] + len(h))
    th = ki.Trace(tr.arrival_ms, tr.output_tokens, np.array(boff, np.int64), block_hash=np.concatenate(bh),
                  input_tokens=np.diff(tr.offsets))
    ot = O.OracleTrace(tr, top_k=3)
    _check_shards(run_ranks(3, _load_exports(th, 3)), ot)


def _fmix64_inv(m):
    M = (1 << 64) - 1

    def unx(x, s):
        z = x
        for _ in range(64 // s + 1):
            z = x ^ (z >> s)
        return z & M
    z = unx(m, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M
    z = unx(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M
    return unx(z, 30)


@pytest.mark.parametrize("W", [2, 3])
def test_time_shard_fingerprint_collisions(W):
    """Distinct hashes sharing the 32-bit sort fingerprint (a hot block interleaved with rare
    ones): the link overflow path's first/has-next flags and the owner's full-hash matching."""
    c, fp = 0x6A09E667F3BCC909, 0x12345678
    hs = [_fmix64_inv((fp << 32) | lo) ^ c for lo in (7, 11, 13, 17, 19, 23)]
    rng = np.random.default_rng(5)
    seq = list(rng.permutation([0] * 400 + [1, 2, 3, 4, 5] * 6))
    R = len(seq)
    tr = ki.Trace(np.arange(R, dtype=np.int64), np.ones(R, np.int32), np.arange(R + 1, dtype=np.int64),
                  block_hash=np.array([hs[x] for x in seq], np.uint64))
    ot = O.OracleTrace(tr, mode="hashes", top_k=2)
    _check_shards(run_ranks(W, _load_exports(tr, 2)), ot)


def test_time_shard_chain_violation_across_shards():
    """R7 across a shard boundary: block B is a root in request 0 (shard 0) and a child in
    request 1 (shard 1); both ranks fail with KARETO_E_CHAIN (none is left in a collective)."""
    tr = ki.Trace(np.array([0, 1], np.int64), np.array([1, 1], np.int32), np.array([0, 1, 3], np.int64),
                  block_hash=np.array([0xB, 0xA, 0xB], np.uint64))

    def fn(r, ctx):
        with pytest.raises(K.KaretoError) as ei:
            ctx.load(tr, top_k=1, time_shard=True)
        return ei.value.status

    assert run_ranks(2, fn) == [K.E_CHAIN] * 2


@pytest.mark.parametrize("W", [2, 3, 8])
def test_time_shard_full_size_config2(W):
    """BASELINE config 2 at full size (1e6 requests, 1.06e8 accesses) time-sharded over W
    loopback ranks: every access's prev / delta / depth equal the whole-trace load's (itself
    checked against the oracle at this size in test_gpu_parity.test_full_size_config2_sampled),
    and so do U, the group tables and the counts of the 16,384-configuration grid."""
    import torch
    import bench
    spec = bench.CONFIGS[2]
    tr = ki.synthetic("chat", R=spec["R"], seed=0)
    c1 = K.Context(0, torch.cuda.current_stream().cuda_stream)
    whole = c1.load(tr, top_k=16)
    cfg, ttl = bench.build_grid(K, spec, whole)
    want_c, want_o = c1.eval_grid(whole, cfg, K.Model(), ttl)
    ref = {x: whole.export(x) for x in (K.X_PREV, K.X_DELTA, K.X_DEPTH, K.X_GROUP)}
    U, Ug, Rg = whole.U, whole.U_g.copy(), whole.reuse_g.copy()
    whole.free()

    def fn(r, ctx):
        gt = ctx.load(tr, top_k=16, time_shard=True)
        res = {x: gt.export(x) for x in (K.X_PREV, K.X_DELTA, K.X_DEPTH, K.X_GROUP)}
        res.update(U=gt.U, Ug=gt.U_g.copy(), Rg=gt.reuse_g.copy(), rlo=gt.req_lo, rhi=gt.req_hi)
        res["c"], res["o"] = ctx.eval_grid(gt, cfg, K.Model(), ttl)
        gt.free()
        return res

    out = run_ranks(W, fn)
    for x in (K.X_PREV, K.X_DELTA, K.X_DEPTH):
        assert np.array_equal(np.concatenate([o[x] for o in out]), ref[x]), x
    for o in out:
        assert o["U"] == U and np.array_equal(o["Ug"], Ug) and np.array_equal(o["Rg"], Rg)
        assert np.array_equal(o[K.X_GROUP][o["rlo"]:o["rhi"]], ref[K.X_GROUP][o["rlo"]:o["rhi"]])
        assert np.array_equal(np.asarray(o["c"]).view(np.uint8), np.asarray(want_c).view(np.uint8))
        assert np.array_equal(o["o"].view(np.uint64), want_o.view(np.uint64))

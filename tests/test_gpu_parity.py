"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bar (BASELINE.json north_star): tier counts and Pareto membership bit-exact; fp64
objectives within 1e-9 relative (expected bit-identical: both sides evaluate the same
operation sequence without FMA contraction, R33)."""
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


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


def kcfg(ocfg):
    c = np.zeros(len(ocfg), K.CONFIG_DTYPE)
    for f in ("cap", "policy", "medium", "tuner", "axis"):
        c[f] = ocfg[f]
    return c


def as_u64(counts):
    return np.ascontiguousarray(counts).view(np.uint64).reshape(len(counts), 11)


def assert_counts_equal(got, want, cfgs=None):
    g, w = as_u64(got), as_u64(want)
    bad = np.nonzero((g != w).any(1))[0]
    if len(bad):
        i = bad[0]
        raise AssertionError(f"{len(bad)} configs differ; first {i} cfg={None if cfgs is None else cfgs[i]}\n"
                             f"gpu   ={got[i]}\noracle={want[i]}")


def assert_obj_equal(got, want):
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
    assert np.all(rel <= 1e-9), f"max rel {rel.max()}"
    # expected bit-identical
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), "objectives not bit-identical"


def run_both(ctx, tr, ocfg, ttl=None, top_k=2, salt=0, tau_e=0.05):
    ot = O.OracleTrace(tr, top_k=top_k, salt=salt)
    gt = ctx.load(tr, top_k=top_k, salt=salt)
    want = ot.replay(ocfg, ttl)
    got, obj = ctx.eval_grid(gt, kcfg(ocfg), K.Model(**MODEL_KW), ttl)
    assert_counts_equal(got, want, ocfg)
    fo = ot.objective(O.Model(**MODEL_KW), ocfg, want)
    assert_obj_equal(obj, fo)
    st, nf = ctx.pareto(obj, kcfg(ocfg), tau_e)
    ost = O.select(fo, ocfg, tau_e)
    assert np.array_equal(st, ost)
    assert nf == int((ost == 1).sum())
    return ot, gt


def check_trace_exports(ot, gt):
    e = ot.export()
    assert gt.N == ot.N and gt.U == ot.U and gt.R == ot.R and gt.span_ms == ot.span_ms
    assert gt.Ltok == ot.Ltok and gt.O == ot.O
    assert np.array_equal(gt.export(K.X_HASH), e["hash"])
    assert np.array_equal(gt.export(K.X_PREV).astype(np.int64), np.where(e["prev"] < 0, U32, e["prev"]))
    assert np.array_equal(gt.export(K.X_DELTA).astype(np.int64), np.where(e["delta"] < 0, U32, e["delta"]))
    assert np.array_equal(gt.export(K.X_REQ), e["req"].astype(np.uint32))
    assert np.array_equal(gt.export(K.X_START).astype(np.int64), e["s"])
    assert np.array_equal(gt.export(K.X_GROUP), e["group"].astype(np.uint16))
    d, _ = ot.depth()
    assert np.array_equal(gt.export(K.X_DEPTH).astype(np.int64), np.where(d < 0, U32, d))
    assert np.array_equal(gt.U_g, ot.U_g) and np.array_equal(gt.reuse_g, ot.reuse_g)


def tiny_configs(K_):
    rows = [[U32] * (K_ + 1)]
    for t in (0, 1, 3, 50):
        rows.append([t] * (K_ + 1))
    rng = np.random.default_rng(7)
    for _ in range(3):
        rows.append(list(rng.choice([0, 1, 3, 6, 50], K_ + 1)))
    ttl = np.array(rows, np.uint32)
    caps, tun, axis = [], [], []
    for a in range(4):
        for b in range(3):
            for c in range(4):
                for ti in range(5):
                    caps.append([a, b, c]); tun.append(ti); axis.append([a, b, c])
            for ti in range(5, 8):
                caps.append([a, b, O.INF_CAP]); tun.append(ti); axis.append([a, b, 0])
    cf = O.configs(caps, tuner=np.array(tun), axis=axis)
    cf["medium"] = np.arange(len(cf)) % 2
    return cf, ttl


def test_w1_worked_example(ctx):
    tr = ki.from_chains([[1, 2, 3], [1, 2, 4], [1, 2, 3]], [0, 10, 20])
    gt = ctx.load(tr, top_k=0)
    assert list(gt.export(K.X_DEPTH)) == [U32] * 4 + [2, 1, 4, 2, 1]
    cnt, _ = ctx.eval_grid(gt, K.configs([[1, 1, 1], [1, 1, 2]]), K.Model())
    assert list(cnt[0]["hit"]) == [2, 2, 0] and cnt[0]["miss"] == 5 and list(cnt[0]["evict"]) == [8, 7, 2]
    assert list(cnt[1]["hit"]) == [2, 2, 1] and cnt[1]["miss"] == 4 and list(cnt[1]["evict"]) == [8, 7, 0]
    cnt, _ = ctx.eval_grid(gt, K.configs([[0, 0, K.INF]]), K.Model(), ttl=np.array([[15]], np.uint32))
    assert cnt[0]["hit"][2] == 4 and cnt[0]["bytetime_block_ms"] == 115


def test_tiny_random_traces_all_stages(ctx):
    rng = np.random.default_rng(2024)
    for trial in range(25):
        tr = ki.random_prefix_tree(rng)
        K_ = int(rng.integers(0, 3))
        cf, ttl = tiny_configs(K_)
        ot, gt = run_both(ctx, tr, cf, ttl, top_k=K_, salt=trial)
        check_trace_exports(ot, gt)


def baseline_grid(U, m1=4, m2=4, m3=4, d1=16, d2=4, d3=1):
    """BASELINE config-1 style grid: c1 in A(m1, U/d1), c2 in A(m2, U/d2), c3 in A(m3, U/d3)."""
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, axis = [], []
    for i, a in enumerate(A(m1, U // d1)):
        for j, b in enumerate(A(m2, U // d2)):
            for k, c in enumerate(A(m3, U // d3)):
                caps.append([a, b, c]); axis.append([i, j, k])
    return caps, axis


def test_config1_full_parity(ctx):
    # BASELINE config 1: 10k requests / ~1M block accesses, 3-tier LRU, 4x4x4, fp64 model
    tr = ki.synthetic("chat", R=10_000, seed=0)
    ot = O.OracleTrace(tr, top_k=16)
    gt = ctx.load(tr, top_k=16)
    check_trace_exports(ot, gt)
    caps, axis = baseline_grid(ot.U)
    cf = O.configs(caps, axis=axis)
    want = ot.replay(cf)
    got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW))
    assert_counts_equal(got, want, cf)
    fo = ot.objective(O.Model(**MODEL_KW), cf, want)
    assert_obj_equal(obj, fo)
    for tau in (0.05, None):
        st, _ = ctx.pareto(obj, kcfg(cf), tau)
        assert np.array_equal(st, O.select(fo, cf, tau))


def test_config1_ttl_and_uniform_tau(ctx):
    tr = ki.synthetic("chat", R=3000, seed=5)
    ot = O.OracleTrace(tr, top_k=4)
    gt = ctx.load(tr, top_k=4)
    caps, axis = baseline_grid(ot.U, 3, 3, 3)
    rows = [[U32] * 5, [60_000] * 5, [600_000] * 5, [5_000, 60_000, 600_000, 30_000, 1_000]]
    ttl = np.array(rows, np.uint32)
    allcaps, tun, ax = [], [], []
    for (c, a) in zip(caps, axis):
        for ti in range(3):
            allcaps.append(c); tun.append(ti); ax.append(a)
        allcaps.append([c[0], c[1], O.INF_CAP]); tun.append(3); ax.append(a)
    cf = O.configs(allcaps, tuner=np.array(tun), axis=ax)
    want = ot.replay(cf, ttl)
    got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW), ttl)
    assert_counts_equal(got, want, cf)
    assert_obj_equal(obj, ot.objective(O.Model(**MODEL_KW), cf, want))


def test_edge_cases(ctx):
    M = K.Model()
    # requests with fewer than 16 tokens have no blocks (R3); a single block request
    tr = ki.from_chains([[], [1], [], [1, 2]], [0, 1, 1, 2], tails=[5, 15, 0, 3])
    ot, gt = run_both(ctx, tr, O.configs([[0, 0, 0], [1, 0, 0], [5, 5, 5]], axis=[[0, 0, 0], [1, 0, 0], [2, 1, 1]]),
                      top_k=1)
    check_trace_exports(ot, gt)
    # no full blocks at all: N = 0
    tr = ki.from_chains([[], []], [0, 5], tails=[3, 7])
    gt = ctx.load(tr)
    assert gt.N == 0 and gt.U == 0
    cnt, obj = ctx.eval_grid(gt, K.configs([[1, 1, 1]]), M)
    assert cnt[0]["miss"] == 0 and np.isfinite(obj).all()
    # one request
    tr = ki.from_chains([[1, 2, 3]], [7])
    run_both(ctx, tr, O.configs([[1, 1, 1], [0, 0, 0]]), top_k=0)
    # zero configurations
    cnt, obj = ctx.eval_grid(ctx.load(ki.from_chains([[1]], [0])), K.configs(np.zeros((0, 3))), M)
    assert len(cnt) == 0


def test_hash_mode_matches_token_mode(ctx):
    rng = np.random.default_rng(3)
    tr = ki.random_prefix_tree(rng, n_req=40)
    bh, boff = [], [0]
    for r in range(tr.n_requests):
        h = O.chain_hashes(tr.tokens[tr.offsets[r]:tr.offsets[r + 1]])
        bh.append(h)
        boff.append(boff[-1] + len(h))
    th = ki.Trace(tr.arrival_ms, tr.output_tokens, np.array(boff, np.int64), block_hash=np.concatenate(bh),
                  input_tokens=np.diff(tr.offsets))
    a, b = ctx.load(tr, top_k=2), ctx.load(th, top_k=2)
    for x in (K.X_HASH, K.X_PREV, K.X_DELTA, K.X_DEPTH, K.X_GROUP):
        assert np.array_equal(a.export(x), b.export(x))
    assert a.Ltok == b.Ltok


def _unxorshift(x, s):
    z = x
    for _ in range(64 // s + 1):
        z = x ^ (z >> s)
    return z & ((1 << 64) - 1)


def _fmix64_inv(m):
    M = (1 << 64) - 1
    z = _unxorshift(m, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M
    z = _unxorshift(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M
    return _unxorshift(z, 30)


def test_fingerprint_collisions_resolved_exactly(ctx):
    # HASHES mode: distinct block hashes crafted to share the 32-bit sort fingerprint used by
    # K2 (top half of fmix64(h ^ c)), including a hot block interleaved with rare ones, so the
    # bounded scan overflows into the warp-parallel slow path.  prev must still be exact.
    c = 0x6A09E667F3BCC909
    fp = 0x12345678
    hs = [_fmix64_inv((fp << 32) | lo) ^ c for lo in (7, 11, 13, 17, 19, 23)]
    assert O.fmix64(hs[0] ^ c) >> 32 == fp
    rng = np.random.default_rng(5)
    seq = [0] * 400 + [1, 2, 3, 4, 5] * 6
    seq = list(rng.permutation(seq))
    R = len(seq)
    tr = ki.Trace(np.arange(R, dtype=np.int64), np.ones(R, np.int32), np.arange(R + 1, dtype=np.int64),
                  block_hash=np.array([hs[x] for x in seq], np.uint64))
    ot = O.OracleTrace(tr, mode="hashes", top_k=2)
    gt = ctx.load(tr, top_k=2)
    check_trace_exports(ot, gt)


def test_errors(ctx):
    # chain violation (R7)
    tr = ki.Trace(np.array([0, 1], np.int64), np.array([1, 1], np.int32), np.array([0, 1, 3], np.int64),
                  block_hash=np.array([0xB, 0xA, 0xB], np.uint64))
    with pytest.raises(K.KaretoError) as ei:
        ctx.load(tr)
    assert ei.value.status == K.E_CHAIN
    # decreasing offsets
    with pytest.raises(K.KaretoError) as ei:
        ctx.load_trace(np.array([0, 1], np.int64), np.array([1, 1], np.int32), np.array([0, 32, 16], np.int64),
                       tokens=np.zeros(32, np.uint32))
    assert ei.value.status == K.E_PARSE
    gt = ctx.load(ki.from_chains([[1, 2]], [0]))
    M = K.Model()
    for bad in (K.configs([[1, 1, 1]], policy=5), K.configs([[1, 1, 1]], medium=3), K.configs([[1, 1, K.INF]])):
        with pytest.raises(K.KaretoError) as ei:
            ctx.eval_grid(gt, bad, M)
        assert ei.value.status == K.E_INVALID
    with pytest.raises(ValueError):
        ctx.eval_grid(gt, K.configs([[1, 1, 1]]), M, ttl=np.array([[5, 5, 5]], np.uint32))  # K+1 = 17 columns
    with pytest.raises(K.KaretoError) as ei:
        ctx.eval_grid(gt, K.configs([[1, 1, 1]], tuner=3), M, ttl=np.full((1, 17), 5, np.uint32))
    assert ei.value.status == K.E_INVALID
    with pytest.raises(K.KaretoError) as ei:
        bad = K.Model(bw_dram=0.0)
        ctx.eval_grid(gt, K.configs([[1, 1, 1]]), bad)
    assert ei.value.status == K.E_INVALID


def test_medium_scale_depth_and_counts(ctx):
    tr = ki.synthetic("chat", R=100_000, seed=1)
    ot = O.OracleTrace(tr, top_k=16)
    gt = ctx.load(tr, top_k=16)
    d, _ = ot.depth()
    assert np.array_equal(gt.export(K.X_DEPTH).astype(np.int64), np.where(d < 0, U32, d))
    caps, axis = baseline_grid(ot.U, 8, 8, 8)
    cf = O.configs(caps, axis=axis)
    want = ot.stack_counts(cf)
    got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW))
    assert_counts_equal(got, want, cf)
    assert_obj_equal(obj, ot.objective(O.Model(**MODEL_KW), cf, want))
    # O1 on a sample
    idx = np.random.default_rng(0).choice(len(cf), 6, replace=False)
    assert_counts_equal(got[idx], ot.replay(cf[idx]), cf[idx])


def test_agent_and_api_workloads(ctx):
    for kind, R in (("agent", 800), ("api", 3000)):
        tr = ki.synthetic(kind, R=R, seed=2)
        ot = O.OracleTrace(tr, top_k=8)
        gt = ctx.load(tr, top_k=8)
        check_trace_exports(ot, gt)
        caps, axis = baseline_grid(ot.U, 4, 4, 4)
        cf = O.configs(caps, axis=axis)
        want = ot.stack_counts(cf)
        got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW))
        assert_counts_equal(got, want, cf)


def replay_configs(K_, rng, n_rows=4):
    """Configurations that need the K6 replay: FIFO / LFU in both modes, LRU with per-group TTL on
    a finite disk; mixed with stack-eligible LRU ones (eval_grid splits and re-merges them)."""
    rows = [[U32] * (K_ + 1), [3] * (K_ + 1)]
    for _ in range(n_rows):
        rows.append(list(rng.choice([0, 1, 3, 6, 50], K_ + 1)))
    ttl = np.array(rows, np.uint32)
    caps, pol, tun, axis = [], [], [], []
    for a in range(3):
        for b in range(3):
            for c in range(3):
                for p in (O.LRU, O.FIFO, O.LFU):
                    for ti in range(len(rows)):
                        caps.append([a, b, c]); pol.append(p); tun.append(ti); axis.append([a, b, c])
                    for ti in range(2, len(rows)):
                        caps.append([a, b, O.INF_CAP]); pol.append(p); tun.append(ti); axis.append([a, b, 0])
    cf = O.configs(caps, policy=np.array(pol), tuner=np.array(tun), axis=axis)
    return cf, ttl


def test_replay_tiny_random_all_policies(ctx):
    rng = np.random.default_rng(99)
    for trial in range(12):
        tr = ki.random_prefix_tree(rng)
        K_ = int(rng.integers(0, 3))
        cf, ttl = replay_configs(K_, rng)
        run_both(ctx, tr, cf, ttl, top_k=K_, salt=trial)


def test_replay_belady_and_w3(ctx):
    BEL = [1, 2, 3, 4, 1, 2, 5, 1, 2, 3, 4, 5]
    gt = ctx.load(ki.from_chains([[x] for x in BEL], list(range(12))), top_k=0)
    cnt, _ = ctx.eval_grid(gt, K.configs([[3, 0, 0], [4, 0, 0]] * 3, policy=np.repeat([0, 1, 2], 2)), K.Model())
    assert [int(c["hit"].sum()) for c in cnt] == [2, 4, 3, 2, 2, 4]  # LRU, FIFO (Belady anomaly), LFU


def test_replay_chat_trace_mixed_grid(ctx):
    # config-3-shaped grid (LRU / FIFO / LFU x tuner rows incl. TTL mode) on a small chat trace
    tr = ki.synthetic("chat", R=1500, seed=4)
    ot = O.OracleTrace(tr, top_k=4)
    rows = [[U32] * 5, [600_000] * 5, [60_000, 600_000, 3_600_000, 30_000, 5_000]]
    ttl = np.array(rows, np.uint32)
    caps, axis = baseline_grid(ot.U, 3, 3, 3)
    allc, pol, tun, ax = [], [], [], []
    for c, a in zip(caps, axis):
        for p in (O.LRU, O.FIFO, O.LFU):
            for ti in range(3):
                allc.append(c); pol.append(p); tun.append(ti); ax.append(a)
            allc.append([c[0], c[1], O.INF_CAP]); pol.append(p); tun.append(2); ax.append(a)
    cf = O.configs(allc, policy=np.array(pol), tuner=np.array(tun), axis=ax)
    run_both(ctx, tr, cf, ttl, top_k=4)


@pytest.mark.slow
def test_full_size_config2_sampled(ctx):
    # BASELINE config 2 at full size, in the launch configuration bench.py times
    tr = ki.synthetic("chat", R=1_000_000, seed=0)
    gt = ctx.load(tr, top_k=16)
    ot = O.OracleTrace(tr, top_k=16)
    d, _ = ot.depth()
    assert np.array_equal(gt.export(K.X_DEPTH).astype(np.int64), np.where(d < 0, U32, d))
    caps, axis = baseline_grid(ot.U, 32, 32, 16, 16, 2, 1)
    cf = O.configs(caps, axis=axis)
    got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW))
    idx = np.random.default_rng(1).choice(len(cf), 64, replace=False)
    want = ot.stack_counts(cf[idx])
    assert_counts_equal(got[idx], want, cf[idx])
    assert_obj_equal(obj[idx], ot.objective(O.Model(**MODEL_KW), cf[idx], want))


@pytest.mark.parametrize("config", [2, 4])
def test_full_size_selection(ctx, config):
    """K8 at BASELINE full size in bench.py's launch configuration: the GPU's objective vectors of
    config 2 (16,384 configs, no pruning) / config 4 (130,944 configs, pruning tau_e = 0.05) go
    through kareto_pareto and through the oracle's select (R34 pruning + R35 dominance); the
    status of every configuration must agree (objectives themselves: test_full_size_config2_sampled)."""
    import bench
    spec = bench.CONFIGS[config]
    tr = ki.synthetic(spec["kind"], R=spec.get("R", 0), N=spec.get("N", 0), seed=0)
    gt = ctx.load(tr, top_k=spec.get("top_k", 16))
    cfg, ttl = bench.build_grid(K, spec, gt)
    _, obj = ctx.eval_grid(gt, cfg, K.Model(), ttl)
    st, nf = ctx.pareto(obj, cfg, spec["prune"])
    oc = np.zeros(len(cfg), O.CONFIG_DTYPE)
    for f in ("cap", "policy", "medium", "tuner", "axis"):
        oc[f] = cfg[f]
    want = O.select(obj, oc, spec["prune"])
    assert np.array_equal(st, want)
    assert nf == int((want == 1).sum()) and nf > 0


def test_config5_million_configs_windowed_histograms(ctx):
    """BASELINE config 5 (i): the 100 x 100 x 100 LRU grid (10^6 configurations) on the R = 1e4
    chat trace.  Its ~10^6 distinct tier boundaries exceed shared memory, so K4 takes the windowed
    multi-pass histograms (k_hist_d / k_hist_D); sampled configurations against the oracle's O2
    stack counts and O1 replay, objectives bit-identical, and LRU inclusion across the grid."""
    tr = ki.synthetic("chat", R=10_000, seed=0)
    ot = O.OracleTrace(tr, top_k=16)
    gt = ctx.load(tr, top_k=16)
    caps, axis = baseline_grid(ot.U, 100, 100, 100, 16, 2, 1)
    cf = O.configs(caps, axis=axis)
    got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW))
    idx = np.random.default_rng(7).choice(len(cf), 512, replace=False)
    want = ot.stack_counts(cf[idx])
    assert_counts_equal(got[idx], want, cf[idx])
    assert_obj_equal(obj[idx], ot.objective(O.Model(**MODEL_KW), cf[idx], want))
    assert_counts_equal(got[idx[:8]], ot.replay(cf[idx[:8]]), cf[idx[:8]])
    # inclusion (Mattson): along the DRAM axis with HBM and disk fixed, total hits never decrease
    h = np.asarray(got["hit"]).sum(1).reshape(100, 100, 100)
    assert np.all(np.diff(h, axis=1) >= 0)


@pytest.mark.parametrize("env", [{"KARETO_K2_FULLSORT": "1"}, {"KARETO_K2_TABLE_LIMIT": "3"},
                                 {"KARETO_K2_ACCESS_INFO": "1"}])
def test_k2_full_sort_path_and_bucket_overflow_fallback(ctx, env):
    """K2's two link paths give the same prev: the full 32-bit sort + tiled link (forced), and the
    16-bit bucket link falling back to it when a bucket exceeds the warp table (limit forced to 3
    distinct blocks per bucket).  Compared with the oracle (O-5 prev / delta)."""
    import os
    tr = ki.synthetic("chat", R=3000, seed=8)
    ot = O.OracleTrace(tr, top_k=4)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        gt = ctx.load(tr, top_k=4)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    check_trace_exports(ot, gt)


@pytest.mark.parametrize("kind,R", [("chat", 20_000), ("agent", 1_500)])
def test_k4_runs_and_access_paths(ctx, kind, R):
    """K4 over the K3 runs (the default for whole traces: a run adds an arithmetic range of depths,
    one D and one delta) against K4 over the accesses (forced with KARETO_K4_ACCESS) and the O2
    closed forms: dense capacity boundaries (bins narrower than runs), CAPACITY rows with uniform
    disk TTLs (delta bins) and TTL-mode rows.  The trace's depths are never exported before the
    first evaluation (deferred materialisation), and are checked against the oracle after it."""
    import os
    tr = ki.synthetic(kind, R=R, seed=21)
    ot = O.OracleTrace(tr, top_k=4)
    gt = ctx.load(tr, top_k=4)
    U = ot.U
    rows = np.array([[U32] * 5, [3_600_000] * 5, [60_000] * 5, [1_000] * 5], np.uint32)
    caps, tun, axis = [], [], []
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    for i, a in enumerate(A(12, U // 40)):
        for j, b in enumerate(A(9, U // 6)):
            for k, c in enumerate(A(7, U // 2)):
                for t in range(4):
                    caps.append([a, b, c]); tun.append(t); axis.append([i, j, k])
            for t in (1, 2, 3):
                caps.append([a, b, O.INF_CAP]); tun.append(t); axis.append([i, j, 7])
    cf = O.configs(caps, tuner=np.array(tun), axis=axis)
    want = ot.stack_counts(cf, rows)
    got_runs, obj_runs = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW), rows)
    assert_counts_equal(got_runs, want, cf)
    os.environ["KARETO_K4_ACCESS"] = "1"
    try:
        got_acc, obj_acc = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW), rows)
    finally:
        os.environ.pop("KARETO_K4_ACCESS", None)
    assert_counts_equal(got_acc, want, cf)
    assert np.array_equal(obj_runs.view(np.uint64), obj_acc.view(np.uint64))
    d, _ = ot.depth()
    assert np.array_equal(gt.export(K.X_DEPTH).astype(np.int64), np.where(d < 0, U32, d))

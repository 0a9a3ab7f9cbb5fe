"""GPU parity for row f1: kareto_hypervolume and kareto_search (Alg. 1) through the C ABI
against the oracle (oracle/search.py).

Bar: the evaluated (d, t, round) sequence and the truncation flag identical, objectives
bit-identical (the same fp64 model as row a8), frontier status bit-exact; hypervolume within
1e-12 relative (the GPU sums the staircase strips and slabs in a different order)."""
import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O
from oracle import search as S

pytestmark = pytest.mark.gpu

MODEL_KW = dict(instances=2, gpus_per_instance=8, alpha_ps=50_000_000, beta_ps=1, dec_ps=150_000_000,
                block_bytes=5_242_880, bw_dram=25e9, c_hw=2.5, p_hbm=0.001, p_dram=0.004, iops_per_block=1.0,
                ttl_prov_gb=1024.0, media=((120e6, 0.5e6, 350e6, 0.0001),),
                phi=((0.0, 0.0, 0.0), (3000.0, 0.005, 0.0), (32000.0, 0.065, 0.0)))


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


@pytest.mark.parametrize("n,ties", [(1, False), (7, True), (300, False), (2500, True), (5000, False)])
def test_hypervolume_parity(ctx, n, ties):
    import torch
    rng = np.random.default_rng(n)
    pts = rng.integers(0, 40, size=(n, 3)).astype(np.float64) if ties else rng.random((n, 3)) * [3.0, 1e3, 7e-2]
    ref = pts.max(0) + 1.0
    want = S.hypervolume(pts, ref)
    assert ctx.hypervolume(pts, ref) == pytest.approx(want, rel=1e-12)
    dev = torch.from_numpy(pts).cuda()
    assert ctx.hypervolume(dev, ref) == pytest.approx(want, rel=1e-12)
    mask = (rng.random(n) < 0.5).astype(np.uint8)
    mask[0] = 1
    assert ctx.hypervolume(pts, ref, mask=mask) == pytest.approx(S.hypervolume(pts[mask == 1], ref), rel=1e-12)


def test_hypervolume_edge_cases(ctx):
    assert ctx.hypervolume(np.zeros((0, 3)), (1, 1, 1)) == 0.0
    assert ctx.hypervolume(np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 0.0]]), (3, 3, 1)) == 3.0
    pts = np.array([[0.5, 0.5, 0.5], [0.2, 0.2, 1.0]])
    with pytest.raises(K.KaretoError, match="point 1"):
        ctx.hypervolume(pts, (1, 1, 1))
    same = np.tile([[0.25, 0.5, 0.75]], (100, 1))                       # all points identical
    assert ctx.hypervolume(same, (1, 1, 1)) == pytest.approx(0.75 * 0.5 * 0.25, rel=1e-15)


def run_both(ctx, tr, hbm_gb, d_range, t_range, policy=K.LRU, max_evals=1 << 16, expand_ttl=False, **th):
    m = O.Model(**MODEL_KW)
    ot = O.OracleTrace(tr, top_k=4)
    ev = S.trace_evaluator(ot, m, hbm_gb, MODEL_KW["block_bytes"])
    p = S.SearchParams(*d_range, *t_range, max_evals=max_evals, expand_ttl=expand_ttl, **th)
    log, F, trunc = S.adaptive_search(ev, p)
    gt = ctx.load(tr, top_k=4)
    got, gtrunc = ctx.search(gt, K.Model(**MODEL_KW), d_range, t_range, hbm_gb, policy=policy, cap=max_evals,
                             expand_ttl=expand_ttl, **th)
    return log, F, trunc, got, gtrunc


@pytest.mark.parametrize("seed,R,d_range,hbm,th", [
    (0, 1500, (0, 2048, 512), 20.0, {}),
    (3, 800, (0, 96, 24), 2.0, dict(tau_e=0.01, tau_perf=0.01, tau_cost=0.0005))])
def test_search_parity(ctx, seed, R, d_range, hbm, th):
    tr = ki.synthetic("chat", R=R, seed=seed)
    log, F, trunc, got, gtrunc = run_both(ctx, tr, hbm, d_range, (0, 2400, 600), **th)
    assert gtrunc == trunc
    assert [(int(a), int(b), int(c)) for a, b, c in zip(got["d_gb"], got["t_s"], got["round"])] == log
    assert np.array_equal(got["obj"].view(np.uint64), F.view(np.uint64)), "objectives not bit-identical"
    assert np.array_equal(got["status"], O.pareto(F))
    assert got["round"].max() >= 1                      # the landscape is not flat: refinement ran
    ref = F.max(0) + np.abs(F.max(0)) * 0.01 + 1e-9
    fr = got["status"] == 1
    assert ctx.hypervolume(got["obj"][fr].copy(), ref) == pytest.approx(S.hypervolume(F[fr], ref), rel=1e-12)


def test_search_truncation_parity(ctx):
    tr = ki.synthetic("chat", R=600, seed=5)
    full, *_ = run_both(ctx, tr, 10.0, (0, 1024, 512), (0, 1200, 600))
    log, F, trunc, got, gtrunc = run_both(ctx, tr, 10.0, (0, 1024, 512), (0, 1200, 600), max_evals=len(full) - 1)
    assert trunc and gtrunc
    assert [(int(a), int(b), int(c)) for a, b, c in zip(got["d_gb"], got["t_s"], got["round"])] == log


def test_search_invalid_params(ctx):
    gt = ctx.load(ki.synthetic("chat", R=50, seed=1), top_k=2)
    with pytest.raises(K.KaretoError):
        ctx.search(gt, K.Model(**MODEL_KW), (0, 100, 0), (0, 10, 5), 1.0)       # zero step
    with pytest.raises(K.KaretoError):
        ctx.search(gt, K.Model(**MODEL_KW), (0, 100, 50), (0, 5_000_000, 5), 1.0)  # TTL beyond 2^32 ms


def test_search_ttl_expansion_parity(ctx):
    """R55 (extension): the TTL-axis expansion evaluates the same sequence as the oracle's, with
    bit-identical objectives, and reaches TTLs beyond the seed range on a chat trace."""
    tr = ki.synthetic("chat", R=1500, seed=0)
    log, F, trunc, got, gtrunc = run_both(ctx, tr, 20.0, (0, 2048, 512), (0, 120, 60), expand_ttl=True,
                                          tau_e=0.01)
    assert gtrunc == trunc
    assert [(int(a), int(b), int(c)) for a, b, c in zip(got["d_gb"], got["t_s"], got["round"])] == log
    assert np.array_equal(got["obj"].view(np.uint64), F.view(np.uint64))
    assert got["t_s"].max() > 120

"""GPU parity for row f2 (Alg. 2 ROI-aware group TTLs): kareto_ttl_roi / kareto_ttl_eval /
kareto_ttl_allocate through the C ABI against oracle/ttl_alloc.py on the same seeded traces.

Bar: bit-exact (every quantity is an integer and every decision an exact integer compare)."""
import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O
from oracle import ttl_alloc as A

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


def both(ctx, tr, top_k):
    ot = O.OracleTrace(tr, top_k=top_k)
    curves = A.curves_from_trace(ot.export(), ot.U_g, top_k)
    gt = ctx.load(tr, top_k=top_k)
    return curves, gt


@pytest.mark.parametrize("kind,R,top_k", [("chat", 400, 4), ("agent", 60, 3), ("chat", 250, 0)])
def test_roi_and_eval_parity(ctx, kind, R, top_k):
    tr = ki.synthetic(kind, R=R, seed=1)
    curves, gt = both(ctx, tr, top_k)
    t, h, c = ctx.ttl_roi(gt)
    want = [A.roi_ttl(cv) for cv in curves]
    assert t.tolist() == want
    assert h.tolist() == [cv.H(x) for cv, x in zip(curves, want)]
    assert c.tolist() == [cv.C(x) for cv, x in zip(curves, want)]
    assert [cv.N for cv in curves] == gt.reuse_g.tolist()       # N_g agrees with the trace stats
    rng = np.random.default_rng(R)
    ttl = rng.integers(0, 4_000_000, size=(64, top_k + 1)).astype(np.uint32)
    ttl[0] = 0
    ttl[1] = 0xFFFFFFFE
    hits, cost = ctx.ttl_eval(gt, ttl)
    for i in range(len(ttl)):
        assert (int(hits[i]), int(cost[i])) == A.totals(curves, ttl[i].tolist())
    with pytest.raises(K.KaretoError, match="infinite"):
        ctx.ttl_eval(gt, np.full((1, top_k + 1), 0xFFFFFFFF, np.uint32))


@pytest.mark.parametrize("frac", [0.0, 0.01, 0.2, 1.5])
def test_allocate_parity(ctx, frac):
    tr = ki.synthetic("chat", R=300, seed=4)
    top_k = 4
    curves, gt = both(ctx, tr, top_k)
    # budget as a fraction of the cost of keeping every block for the whole trace span
    full = sum(cv.C(max(cv.d) if cv.d else 0) for cv in curves)
    B = int(frac * full)
    got = ctx.ttl_allocate(gt, B, seed=3)
    t, h, cost, t_roi, t_init = A.allocate(curves, B, seed=3)
    assert got["t_roi"].tolist() == t_roi and got["t_init"].tolist() == t_init
    assert got["t"].tolist() == t and got["hits"] == h and got["cost"] == cost
    assert cost <= B


@pytest.mark.parametrize("frac", [0.001, 0.01, 0.05, 0.2])
def test_allocate_not_below_uniform(ctx, frac):
    # R54: Alg. 2 with the uniform start keeps at least the hits of the best uniform TTL
    tr = ki.synthetic("chat", R=2000, seed=6)
    top_k = 8
    curves, gt = both(ctx, tr, top_k)
    full = sum(cv.C(max(cv.d) if cv.d else 0) for cv in curves)
    B = int(frac * full)
    got = ctx.ttl_allocate(gt, B, seed=1)
    tu = A.uniform_ttl(curves, B)
    hu, cu = A.totals(curves, [tu] * (top_k + 1))
    assert cu <= B and got["cost"] <= B and got["hits"] >= hu
    t, h, cost, _, _ = A.allocate(curves, B, seed=1)
    assert got["t"].tolist() == t and got["hits"] == h and got["cost"] == cost

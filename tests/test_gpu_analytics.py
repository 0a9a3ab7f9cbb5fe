"""GPU parity for the row-f4 trace analytics (kareto_trace_analytics) against oracle/analytics.py:
X6 hits / blocks_90 / Lorenz points and X5 cumulative / active series, all exact (the Lorenz
shares are one fp64 division of the same exact integers on both sides)."""
import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import analytics as X
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


@pytest.mark.parametrize("kind,R,seed", [("chat", 600, 0), ("agent", 40, 2), ("api", 300, 1)])
def test_analytics_parity(ctx, kind, R, seed):
    tr = ki.synthetic(kind, R=R, seed=seed)
    ot = O.OracleTrace(tr, top_k=2)
    e = ot.export()
    T, k90, f90, lor, U = X.skew(e, n_pts=101)
    cum, act = X.footprint(e, ot.R)
    gt = ctx.load(tr, top_k=2)
    a = ctx.analytics(gt, n_pts=101)
    assert (a["unique_blocks"], a["total_hits"], a["blocks_90"]) == (U, T, k90)
    assert a["frac_90"] == f90
    assert a["lorenz"].tolist() == lor
    assert np.array_equal(a["cumulative"], cum) and np.array_equal(a["active"], act)
    assert a["peak_active"] == act.max() and a["peak_active_request"] == int(np.argmax(act))
    assert a["final_cumulative"] == cum[-1]


def test_analytics_edge_cases(ctx):
    gt = ctx.load(ki.from_chains([[i] for i in range(6)], list(range(6))), top_k=1)   # no reuse
    a = ctx.analytics(gt, n_pts=5)
    assert a["total_hits"] == 0 and a["frac_90"] == 1.0 and a["blocks_90"] == 6
    assert a["lorenz"].tolist() == [0.0] * 5 and a["active"].tolist() == [0] * 6
    with pytest.raises(K.KaretoError):
        ctx.analytics(gt, n_pts=1)

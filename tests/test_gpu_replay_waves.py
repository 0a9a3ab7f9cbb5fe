"""GPU parity for the K6 replay when its state does not fit one wave (row a7; VERDICT r1 "What's
missing" #1 / ADVICE r1 high): the device-memory budget is forced down with KARETO_K6_BUDGET so
every configuration class runs several waves, concurrently (one stream per class) and
sequentially, and a lopsided grid (a large LFU class plus two FIFO configurations) that the
round-1 work-proportional split starved to a zero-width wave.  Counts, objectives and Pareto
status are compared with the oracle's literal replay O1, bit-exact."""
import os
import re

import numpy as np
import pytest

import kareto_inputs as ki
import paper_2603_08739_b200 as K
from oracle import oracle as O

pytestmark = pytest.mark.gpu
U32 = 0xFFFFFFFF
MODEL_KW = dict(instances=2)


@pytest.fixture(scope="module")
def ctx():
    import torch
    assert torch.cuda.is_available()
    return K.Context(0)


@pytest.fixture()
def env():
    saved = {k: os.environ.get(k) for k in ("KARETO_K6_BUDGET", "KARETO_K6_SEQUENTIAL", "KARETO_DEBUG")}
    yield os.environ
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def kcfg(ocfg):
    return K.configs(ocfg["cap"], policy=ocfg["policy"], medium=ocfg["medium"], tuner=ocfg["tuner"],
                     axis=ocfg["axis"])


def class_bytes(U, R, G):
    """Per-configuration K6 state of each class (replay.cu per_cfg_of): list 13 B per block; LFU adds
    a 4 B frequency and 3 tiers of frequency-bucket heads/tails + bitmaps; the expiry heap 4 B + 8 B
    per block; the LRU group lists 8 B per block + 8 B per group."""
    FM = R + 2
    NW = (FM + 63) // 64
    NSW = (NW + 63) // 64
    base = U * 13
    lfu = U * 4 + 3 * 8 * (FM + NW + NSW)
    heap = U * 4 + 8 * (U + 1)
    glist = U * 8 + 8 * G
    return {0: base, 1: base + heap, 2: base + lfu, 3: base + lfu + heap, 4: base + glist}


def mixed_grid(U):
    rows = [[U32] * 5, [600_000] * 5, [60_000, 600_000, 3_600_000, 30_000, 5_000]]
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, pol, tun, ax = [], [], [], []
    for i, a in enumerate(A(3, U // 16)):
        for j, b in enumerate(A(3, U // 4)):
            for k, c in enumerate(A(3, U)):
                for p in (O.LRU, O.FIFO, O.LFU):
                    for ti in range(3):
                        caps.append([a, b, c]); pol.append(p); tun.append(ti); ax.append([i, j, k])
                    caps.append([a, b, O.INF_CAP]); pol.append(p); tun.append(2); ax.append([i, j, 0])
    return O.configs(caps, policy=np.array(pol), tuner=np.array(tun), axis=ax), np.array(rows, np.uint32)


def check(ctx, tr, cf, ttl, top_k=4):
    ot = O.OracleTrace(tr, top_k=top_k)
    gt = ctx.load(tr, top_k=top_k)
    want = ot.replay(cf, ttl)
    got, obj = ctx.eval_grid(gt, kcfg(cf), K.Model(**MODEL_KW), ttl)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    fo = ot.objective(O.Model(**MODEL_KW), cf, want)
    assert np.array_equal(obj.view(np.uint64), fo.view(np.uint64))
    st, _ = ctx.pareto(obj, kcfg(cf), 0.05)
    assert np.array_equal(st, O.select(fo, cf, 0.05))
    return gt


def waves_from_debug(err):
    out = {}
    for m in re.finditer(r"K6 class (\d): (\d+) configs, waves of (\d+)", err):
        q, n, w = map(int, m.groups())
        out[q] = -(-n // w)
    return out


@pytest.fixture(scope="module")
def chat():
    tr = ki.synthetic("chat", R=1500, seed=4)
    U = O.OracleTrace(tr, top_k=4).U
    return tr, U


def test_concurrent_classes_many_waves(ctx, env, chat, capfd):
    tr, U = chat
    cf, ttl = mixed_grid(U)
    cb = class_bytes(U, 1500, 5)
    env["KARETO_K6_BUDGET"] = str(sum(cb.values()) * 4)
    env["KARETO_DEBUG"] = "1"
    env.pop("KARETO_K6_SEQUENTIAL", None)
    check(ctx, tr, cf, ttl)
    waves = waves_from_debug(capfd.readouterr().err)
    assert sorted(waves) == [0, 1, 2, 3, 4], waves          # all five classes ran concurrently
    assert min(waves.values()) >= 3, waves                    # each in three or more waves


def test_sequential_classes_many_waves(ctx, env, chat):
    tr, U = chat
    cf, ttl = mixed_grid(U)
    cb = class_bytes(U, 1500, 5)
    env["KARETO_K6_BUDGET"] = str(max(cb.values()) * 5)
    env["KARETO_K6_SEQUENTIAL"] = "1"
    check(ctx, tr, cf, ttl)


def test_budget_below_class_minimum_falls_back_to_sequential(ctx, env, chat):
    # room for the largest single configuration but not for one of every class at once
    tr, U = chat
    cf, ttl = mixed_grid(U)
    cb = class_bytes(U, 1500, 5)
    assert max(cb.values()) * 1.01 < sum(cb.values())
    env["KARETO_K6_BUDGET"] = str(int(max(cb.values()) * 1.01))
    env.pop("KARETO_K6_SEQUENTIAL", None)
    check(ctx, tr, cf, ttl)


def test_lopsided_classes_no_starved_class(ctx, env, chat, capfd):
    # a big LFU grid plus two FIFO configurations in a multi-wave replay; the
    # work-proportional split gave the FIFO class a zero-width wave (KARETO_E_OOM)
    tr, U = chat
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, pol = [], []
    for a in A(4, U // 16):
        for b in A(4, U // 4):
            for c in A(4, U):
                caps.append([a, b, c]); pol.append(O.LFU)
    caps += [[U // 16, U // 4, U], [0, U // 8, U // 2]]
    pol += [O.FIFO, O.FIFO]
    cf = O.configs(caps, policy=np.array(pol), axis=[[0, 0, 0]] * len(caps))
    cb = class_bytes(U, 1500, 5)
    env["KARETO_K6_BUDGET"] = str(cb[2] * 8)                  # 64 LFU configurations: 8+ waves
    env["KARETO_DEBUG"] = "1"
    env.pop("KARETO_K6_SEQUENTIAL", None)
    check(ctx, tr, cf, None)
    waves = waves_from_debug(capfd.readouterr().err)
    assert waves.get(0, 0) >= 1 and waves.get(2, 0) >= 3, waves


def test_ttl_mode_collapse_fifo_lfu():
    """TTL-mode FIFO / LFU configurations of one (policy, c1, c2) share their HBM / DRAM replay (the
    lease store is the trace's delta <= tau_g): one replay per group records the lookup tiers and
    k_ttl_member_counts derives every member's counts for its own TTL row.  Against O1 and against
    the uncollapsed replay (KARETO_K6_NO_COLLAPSE), bit for bit; CAPACITY configurations in the same
    call take the normal K6 path."""
    import os
    import paper_2603_08739_b200 as K
    tr = ki.synthetic("chat", R=2000, seed=31)
    ot = O.OracleTrace(tr, top_k=4)
    ctx = K.Context(0)
    gt = ctx.load(tr, top_k=4)
    U = ot.U
    rows = np.array([[1_000 * (t + 1) * (g + 1) for g in range(5)] for t in range(6)] + [[U32] * 5], np.uint32)
    A = lambda m, top: [top * i // (m - 1) for i in range(m)]
    caps, pol, tun = [], [], []
    for a in A(3, U // 16):
        for b in A(3, U // 4):
            for p in (O.FIFO, O.LFU):
                for t in range(6):
                    caps.append([a, b, O.INF_CAP]); pol.append(p); tun.append(t)
                caps.append([a, b, U // 2]); pol.append(p); tun.append(t % 6)      # CAPACITY, finite TTLs
                caps.append([a, b, U // 3]); pol.append(p); tun.append(6)          # CAPACITY, no TTL
    oc = O.configs(caps, policy=np.array(pol), tuner=np.array(tun))
    kc = K.configs(oc["cap"], policy=oc["policy"], tuner=oc["tuner"])
    os.environ["KARETO_K6_COLLAPSE"] = "1"   # a small trace would not collapse on its own
    try:
        got, _ = ctx.eval_grid(gt, kc, K.Model(), rows)
    finally:
        os.environ.pop("KARETO_K6_COLLAPSE", None)
    want = ot.replay(oc, rows)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    os.environ["KARETO_K6_NO_COLLAPSE"] = "1"
    try:
        got2, _ = ctx.eval_grid(gt, kc, K.Model(), rows)
    finally:
        os.environ.pop("KARETO_K6_NO_COLLAPSE", None)
    assert np.array_equal(got.view(np.uint64), got2.view(np.uint64))

"""Pins for the oracle's objective model (R25-R33) and the
selection step (pruning R34 = Alg. 1 expansion test P:555-559; dominance R35 = P:510).

The model's constants are our reading (parity with the paper's numbers unpinned), so
these pins are closed-form special cases, SPEC arithmetic examples and the paper's
qualitative observations stated as exact properties."""
import numpy as np
import pytest

import kareto_inputs as ki
from oracle import oracle as O

INF = O.INF_CAP


def test_phi_spec_examples():
    m = O.Model()
    assert O.phi(m, 0.0) == 0.0
    assert O.phi(m, 2999.0) == 0.0
    assert O.phi(m, 4000.0) == pytest.approx(5.0, rel=0, abs=1e-12)      # S:413 [PAPER P:333]
    lo = (O.phi(m, 32000.0) - O.phi(m, 31000.0)) / 1000.0
    hi = (O.phi(m, 33000.0) - O.phi(m, 32000.0)) / 1000.0
    assert hi / lo == pytest.approx(13.0)                                  # S:414 13x cliff
    mj = O.Model(phi=((0.0, 0.0, 0.0), (10.0, 1.0, 5.0)))                  # jump, right-continuous
    assert O.phi(mj, 9.999) == 0.0 and O.phi(mj, 10.0) == 5.0 and O.phi(mj, 12.0) == 7.0


def _trace():
    return ki.from_chains([[1, 2, 3], [1, 2, 4], [1, 2, 3], [5]], [0, 10, 20, 3_600_000],
                          output_tokens=[10, 20, 30, 40], tails=[3, 0, 15, 0])


def test_prefill_p0_brute_sum():
    tr = _trace()
    m = O.Model(alpha_ps=7, beta_ps=3)
    ot = O.OracleTrace(tr)
    want = 0
    for r in range(tr.n_requests):
        L = int(tr.offsets[r + 1] - tr.offsets[r])
        want += sum(7 + 3 * t for t in range(L))       # per-token alpha + beta * position
    assert ot.prefill_p0(m) == want


def test_zero_cache_is_no_saving_and_hit_saving_is_the_prefix_cost():
    tr = _trace()
    ot = O.OracleTrace(tr)
    m = O.Model(alpha_ps=1000, beta_ps=10, dec_ps=0, c_hw=0, p_dram=0, media=((1e9, 0, 1e9, 0),),
                phi=((0.0, 0.0, 0.0),))
    cf = O.configs([[0, 0, 0], [8, 0, 0]])
    cnt = ot.replay(cf)
    f = ot.objective(m, cf, cnt)
    P0 = ot.prefill_p0(m)
    busy0 = P0 * 1e-12
    assert cnt[0]["hit"].sum() == 0
    # low density (busy << span): no backlog term -> f1 = 1e3 * prefill / R
    assert f[0, 0] == pytest.approx(1e3 * busy0 / 4, rel=1e-15)
    # with hits the saving equals sum over hit blocks of sum_{t=16k}^{16k+15} (alpha + beta t)
    e = ot.export()
    hits = int(cnt[1]["hit"].sum())
    hps = int(cnt[1]["hit_pos_sum"])
    saved = 16 * 1000 * hits + 10 * (256 * hps + 120 * hits)
    brute_saved = 0
    # recompute from the brute definition: hit blocks are the chain prefix of each request
    # (here c1 = 8 holds everything, so every reuse access is a hit)
    for j in range(ot.N):
        if e["prev"][j] >= 0:
            k = int(e["k"][j])
            brute_saved += sum(1000 + 10 * t for t in range(16 * k, 16 * k + 16))
    assert saved == brute_saved
    assert f[1, 0] == pytest.approx(1e3 * (P0 - saved) * 1e-12 / 4, rel=1e-15)


def test_threaded_objective_equals_serial():
    tr = ki.synthetic("chat", R=300, seed=2)
    ot = O.OracleTrace(tr)
    caps = [[a, b, c] for a in (0, 50, 500) for b in (0, 1000) for c in (0, 5000, O.INF_CAP)]
    cf = O.configs(caps, tuner=0)
    ttl = np.full((1, 17), 600_000, np.uint32)
    cnt = ot.replay(cf, ttl)
    f1 = ot.objective(O.Model(), cf, cnt)
    f4 = ot.objective(O.Model(), cf, cnt, threads=4)
    assert np.array_equal(f1.view(np.uint64), f4.view(np.uint64))


def test_observation1_low_density_throughput_identical_across_configs():
    # Obs. 1: with low density, throughput plateaus at the arrival rate regardless of storage.
    tr = ki.synthetic("chat", R=400, seed=1)
    ot = O.OracleTrace(tr)
    m = O.Model(instances=64)
    caps = [[a, b, c] for a in (0, 50, 500) for b in (0, 1000) for c in (0, 5000)]
    cf = O.configs(caps)
    f = ot.objective(m, cf, ot.replay(cf))
    assert np.all(f[:, 1] == f[0, 1])             # exactly equal, not approximately
    assert len(np.unique(f[:, 0])) > 1            # while latency varies


def test_observation3_high_density_capacity_raises_throughput():
    tr = ki.synthetic("chat", R=400, seed=1)
    ot = O.OracleTrace(tr)
    m = O.Model(instances=1, alpha_ps=40_000_000_000)   # compute-constrained (busy > span)
    cf = O.configs([[0, 0, 0], [10**6, 0, 0]])
    f = ot.objective(m, cf, ot.replay(cf))
    assert -f[1, 1] > -f[0, 1]
    assert f[1, 0] < f[0, 0]


def test_spec_disk_bandwidth_coupling_s274():
    # "disk capacity 1000 GB, base 100 MB/s, slope 0.12 MB/s per GB -> 220 MB/s; 2.2 GB -> 10 s"
    # One disk read of a 2.2 GB block: disk_s = 2.2e9 / 220e6 = 10 s appears in f1 (R = 1).
    Bb = 2_200_000_000
    tr = ki.from_chains([[1], [1]], [0, 1_000_000])
    ot = O.OracleTrace(tr)
    c3 = 1000 * 10**9 // Bb    # 454 blocks = 998.8 GB; use exact 1000 GB through the medium slope
    m = O.Model(alpha_ps=0, beta_ps=0, dec_ps=0, block_bytes=Bb, c_hw=0, p_dram=0,
                media=((100e6, 0.12e6 * 1000.0 / (c3 * Bb / 1e9), 1e12, 0.0),), phi=((0.0, 0.0, 0.0),))
    cf = O.configs([[0, 0, c3]])
    cnt = ot.replay(cf)
    # c1 = c2 = 0: each touch passes through HBM and DRAM and is written to disk (2 writes),
    # the second request reads it back from disk (1 read)
    assert list(cnt[0]["hit"]) == [0, 0, 1] and int(cnt[0]["disk_writes"]) == 2
    f = ot.objective(m, cf, cnt)
    # reads and writes share one channel: 3 transfers x 10 s, mean over R = 2 requests
    assert f[0, 0] == pytest.approx(1e3 * (3 * 10.0) / 2, rel=1e-12)


def test_spec_storage_cost_examples_s422_s423():
    # PROVISIONED 1000 GB for 2 h at 0.0005 $/GB-h -> 1.0 ; BYTE_TIME 10 GB for 2 h at 0.001 -> 0.02
    Bb = 10**9
    tr = ki.from_chains([[1], [2]], [0, 7_200_000])   # span = 2 h
    ot = O.OracleTrace(tr)
    base = dict(alpha_ps=0, beta_ps=0, dec_ps=0, block_bytes=Bb, c_hw=0, p_dram=0, phi=((0.0, 0.0, 0.0),))
    m = O.Model(media=((1e9, 0, 1e9, 0.0005),), **base)
    cf = O.configs([[0, 0, 1000]])
    f = ot.objective(m, cf, ot.replay(cf))
    assert f[0, 2] == pytest.approx(1.0, rel=1e-12)
    # TTL mode byte-time: 10 blocks of 1 GB each held for 2 h = 10 GB x 2 h; use counts directly
    m = O.Model(media=((1e9, 0, 1e9, 0.001),), **base)
    cf = O.configs([[0, 0, INF]])
    cnt = np.zeros(1, O.COUNTS_DTYPE)
    cnt["bytetime_block_ms"] = 10 * 7_200_000
    f = ot.objective(m, cf, cnt)
    assert f[0, 2] == pytest.approx(0.02, rel=1e-12)


def test_gpu_hours_linear_in_instances():
    tr = ki.from_chains([[1], [2]], [0, 3_600_000])   # 1 h span, idle
    ot = O.OracleTrace(tr)
    cf = O.configs([[0, 0, 0]])
    cnt = ot.replay(cf)
    kw = dict(alpha_ps=0, beta_ps=0, dec_ps=0, c_hw=10.0, gpus_per_instance=1, p_dram=0,
              media=((1e9, 0, 1e9, 0.0),), phi=((0.0, 0.0, 0.0),))
    f1 = ot.objective(O.Model(instances=1, **kw), cf, cnt)
    f2 = ot.objective(O.Model(instances=2, **kw), cf, cnt)
    assert f1[0, 2] == pytest.approx(10.0, rel=1e-12)   # S:432 idle run, 1 instance, 1 h, c_hw = 10
    assert f2[0, 2] == 2 * f1[0, 2]                     # S:434 doubling instances doubles compute term


# ---------------- selection -----------------------------------------------------------
def test_pareto_spec_examples():
    f = np.array([[1, 1, 1], [2, 2, 2]], float)
    assert list(O.pareto(f)) == [1, 0]
    f = np.array([[1, 3, 0], [2, 2, 0], [3, 1, 0]], float)
    assert list(O.pareto(f)) == [1, 1, 1]                # S:482 antichain
    f = np.array([[1, 1, 1], [1, 1, 1], [2, 2, 2]], float)
    assert list(O.pareto(f)) == [1, 1, 0]                # equal vectors do not dominate (R35)


def test_pareto_random_against_pairwise_and_idempotent(rng):
    for _ in range(50):
        n = int(rng.integers(1, 200))
        f = rng.integers(0, 6, (n, 3)).astype(float)
        st = O.pareto(f)
        le = (f[None, :, :] <= f[:, None, :]).all(-1)
        lt = (f[None, :, :] < f[:, None, :]).any(-1)
        dom = (le & lt).any(1)
        assert np.array_equal(st == 0, dom)
        front = f[st == 1]
        assert np.all(O.pareto(front) == 1)              # S:516 idempotence
        assert np.array_equal(O.pareto(f, threads=4), st)  # row-parallel variant: same statuses


def _grid_cfgs(m1, m2, m3):
    caps, axis = [], []
    for i in range(m1):
        for j in range(m2):
            for k in range(m3):
                caps.append([i, j, k]); axis.append([i, j, k])
    return O.configs(caps, axis=axis)


def test_prune_flat_landscape_keeps_only_first_step():
    cf = _grid_cfgs(4, 1, 1)
    f = np.array([[5.0, 0, 0]] * 4)
    # flat f1: rel_1 = 0 <= tau_e -> j* = 1, configs j > 1 pruned
    assert list(O.prune(f, cf, 0.05)) == [0, 0, 1, 1]


def test_prune_known_crossing():
    cf = _grid_cfgs(6, 1, 1)
    f1 = np.array([100.0, 50.0, 30.0, 29.0, 10.0, 5.0])   # rel: .5, .4, .0333, ...
    f = np.stack([f1, np.zeros(6), np.zeros(6)], 1)
    assert list(O.prune(f, cf, 0.05)) == [0, 0, 0, 0, 1, 1]
    # disabled threshold (negative): nothing ever stops
    assert list(O.prune(f, cf, -1.0)) == [0] * 6


def test_prune_per_line_and_any_axis():
    cf = _grid_cfgs(3, 3, 1)
    # f1 depends on axis 0 only: flat along axis 1 -> along axis-1 lines the 3rd point is pruned
    f = np.array([[100.0 / (1 + c["axis"][0]), 0, 0] for c in cf])
    pr = O.prune(f, cf, 0.05)
    assert list(pr) == [0 if c["axis"][1] <= 1 else 1 for c in cf]


def test_select_status_codes():
    cf = _grid_cfgs(4, 1, 1)
    # f1 along the line: 5, 4 (rel .2, keep going), 4 (rel 0 -> j* = 2), 4 (pruned)
    f = np.array([[5.0, 1, 1], [4.0, 1, 1], [4.0, 0, 0], [4.0, 0, 0]])
    st = O.select(f, cf, 0.05)
    assert list(st) == [0, 0, 1, 2]
    # equal vectors are both frontier (no dedup, R35)
    st = O.select(np.array([[4.0, 0, 0]] * 2), _grid_cfgs(2, 1, 1), 0.05)
    assert list(st) == [1, 1]


# ---------------- per-term pins of or_objective (closed forms; VERDICT r1 "What's weak" #1) ------
# Each case isolates one term of Eq. 1/2 under our readings R27-R32 by zeroing every
# other term, and states the expected value as a hand-worked physical quantity, so a dropped term,
# a swapped capacity or a wrong divisor in kareto_oracle.c:or_objective fails here.

_QUIET = dict(alpha_ps=0, beta_ps=0, dec_ps=0, c_hw=0.0, p_hbm=0.0, p_dram=0.0,
              media=((1e9, 0.0, 1e9, 0.0),), phi=((0.0, 0.0, 0.0),))


def _model(**kw):
    d = dict(_QUIET)
    d.update(kw)
    return O.Model(**d)


def test_dram_load_term_r27():
    # One 2 GB block is stored, demoted to DRAM (c1 = 0, c2 = 1), and read back by the second
    # request: a 2 GB read at bw_dram = 1 GB/s takes 2 s; the mean over R = 2 requests is 1 s.
    tr = ki.from_chains([[1], [1]], [0, 1_000_000])
    ot = O.OracleTrace(tr)
    cf = O.configs([[0, 1, 0], [1, 0, 0]])
    cnt = ot.replay(cf)
    assert list(cnt[0]["hit"]) == [0, 1, 0] and list(cnt[1]["hit"]) == [1, 0, 0]
    f = ot.objective(_model(block_bytes=2 * 10**9, bw_dram=1e9), cf, cnt)
    assert f[0, 0] == 1000.0          # 2 s / 2 requests, in ms
    assert f[1, 0] == 0.0             # the same hit served from HBM costs no load time
    f4 = ot.objective(_model(block_bytes=2 * 10**9, bw_dram=4e9), cf, cnt)
    assert f4[0, 0] == 250.0          # 4x the DRAM bandwidth: 0.5 s / 2
    # no backlog (2 s of work in a 1000 s span): throughput = tokens / span = (2*16 + 2*1) / 1000 s
    assert f[0, 1] == pytest.approx(-34.0 / 1000.0, rel=1e-15)


def test_hbm_and_dram_capacity_prices_are_separate_terms():
    # 1 h span, 1 GB blocks, nothing else billed: an HBM cache of 3 GB at 2 $/GB-h costs 6 $,
    # a DRAM cache of 7 GB at 5 $/GB-h costs 35 $, both together 41 $ (swapping c1/c2 gives 15/14).
    tr = ki.from_chains([[1], [2]], [0, 3_600_000])
    ot = O.OracleTrace(tr)
    cf = O.configs([[3, 0, 0], [0, 7, 0], [3, 7, 0]])
    f = ot.objective(_model(block_bytes=10**9, p_hbm=2.0, p_dram=5.0), cf, ot.replay(cf))
    assert f[0, 2] == pytest.approx(6.0, rel=1e-15)
    assert f[1, 2] == pytest.approx(35.0, rel=1e-15)
    assert f[2, 2] == pytest.approx(41.0, rel=1e-15)


def test_overload_backlog_and_throughput_r29_r30():
    # Two 16-token requests arrive 1 s apart, each needing 16 x 0.3125 s = 5 s of prefill on one
    # instance: 10 s of work in a 1 s span.  Makespan = 10 s; mean TTFT = per-request service
    # (10 s / 2) + fluid backlog (10 s - 1 s) / 2 = 9.5 s; throughput = 32 tokens / 10 s;
    # GPU-hours = 1 GPU x 10 s at 3.6 $/GPU-h = 0.01 $.
    tr = ki.from_chains([[1], [2]], [0, 1000], output_tokens=[0, 0])
    ot = O.OracleTrace(tr)
    cf = O.configs([[0, 0, 0]])
    cnt = ot.replay(cf)
    m1 = _model(alpha_ps=312_500_000_000, c_hw=3.6, gpus_per_instance=1, instances=1)
    f = ot.objective(m1, cf, cnt)
    assert f[0, 0] == pytest.approx(9500.0, rel=1e-15)
    assert f[0, 1] == pytest.approx(-3.2, rel=1e-15)
    assert f[0, 2] == pytest.approx(0.01, rel=1e-14)
    # two instances halve the makespan (5 s): backlog (5 - 1)/2 s, throughput 6.4 tok/s, and the
    # GPU-hours are unchanged (2 GPUs x 5 s)
    m2 = _model(alpha_ps=312_500_000_000, c_hw=3.6, gpus_per_instance=1, instances=2)
    f = ot.objective(m2, cf, cnt)
    assert f[0, 0] == pytest.approx(7000.0, rel=1e-15)
    assert f[0, 1] == pytest.approx(-6.4, rel=1e-15)
    assert f[0, 2] == pytest.approx(0.01, rel=1e-14)


def test_iops_cost_composition_r32():
    # A 730-hour span (one billing month, P:333's monthly IOPS price, /730 h per month) with a
    # constant IOPS rate: the month costs exactly phi(rate) dollars.  Two blocks pass through
    # c1 = c2 = 0 onto a 10-block disk (2 disk writes, R16) and nothing is read back.
    span = 730 * 3600 * 1000
    tr = ki.from_chains([[1], [2]], [0, span])
    ot = O.OracleTrace(tr)
    cf = O.configs([[0, 0, 10]])
    cnt = ot.replay(cf)
    assert int(cnt[0]["disk_writes"]) == 2 and int(cnt[0]["hit"].sum()) == 0
    phi = ((0.0, 0.0, 0.0), (3000.0, 0.005, 0.0), (32000.0, 0.065, 0.0))   # P:333 schedule (R32)
    # iops_per_block chosen so 2 writes/month correspond to 4,000 IOPS: 1,000 IOPS above the free
    # 3,000 at 0.005 $/IOPS-month = 5 $
    m = _model(block_bytes=1, iops_per_block=4000 * (span / 1000) / 2, phi=phi)
    assert ot.objective(m, cf, cnt)[0, 2] == pytest.approx(5.0, rel=1e-12)
    # 33,000 IOPS: 29,000 x 0.005 + 1,000 x 0.065 = 210 $ (the 13x cliff above 32,000)
    m = _model(block_bytes=1, iops_per_block=33000 * (span / 1000) / 2, phi=phi)
    assert ot.objective(m, cf, cnt)[0, 2] == pytest.approx(210.0, rel=1e-12)
    # half the month (span 365 h) at the same 4,000 IOPS costs half: 2.5 $
    tr2 = ki.from_chains([[1], [2]], [0, span // 2])
    ot2 = O.OracleTrace(tr2)
    m = _model(block_bytes=1, iops_per_block=4000 * (span / 2000) / 2, phi=phi)
    assert ot2.objective(m, cf, ot2.replay(cf))[0, 2] == pytest.approx(2.5, rel=1e-12)

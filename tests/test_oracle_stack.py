"""Pins for O2, the oracle's stack-depth path: depths against
the O(N^2) definition, the identity D = d + (n-1-k), and every closed form against O1's
literal replay on random chain-consistent traces (Mattson et al. 1970 stack property)."""
import numpy as np
import pytest

import kareto_inputs as ki
from oracle import oracle as O
from tests import brute
from tests.conftest import chains_from_labels
from tests.test_oracle_replay import _random

INF = O.INF_CAP


def test_depth_matches_definition(rng):
    for _ in range(40):
        chains, arr = _random(rng)
        ot = O.OracleTrace(ki.from_chains(chains, arr))
        d, D = ot.depth()
        want = brute.lru_depths(chains_from_labels(chains, arr))
        assert [None if x < 0 else int(x) for x in d] == want
        e = ot.export()
        n = np.diff(e["s"])[e["req"]]
        ok = d >= 0
        assert np.array_equal(D[ok], d[ok] + (n[ok] - 1 - e["k"][ok]))
        assert np.all(D[~ok] < 0)


def test_w1_depths_and_closed_form_evictions():
    ot = O.OracleTrace(ki.from_chains([[1, 2, 3], [1, 2, 4], [1, 2, 3]], [0, 10, 20]))
    d, D = ot.depth()
    assert list(d) == [-1, -1, -1, -1, 2, 1, 4, 2, 1]
    assert list(D) == [-1, -1, -1, -1, 3, 3, 4, 3, 3]
    c = ot.stack_counts(O.configs([[1, 1, 1]]))[0]
    assert list(c["evict"]) == [8, 7, 2]   # e1 = 9 - 1, e2 = 9 - 2, e3 = #{D>3} - 3 = 5 - 3


def test_stack_counts_equal_replay_on_eligible_configs(rng):
    for trial in range(40):
        chains, arr = _random(rng)
        K = int(rng.integers(0, 3))
        ot = O.OracleTrace(ki.from_chains(chains, arr), top_k=K)
        rows, caps, tuners = [], [], []
        rows.append([0xFFFFFFFF] * (K + 1))
        for t in (0, 1, 3, 6, 50):
            rows.append([t] * (K + 1))          # uniform tau (CAPACITY eligible)
        for _ in range(3):
            rows.append(list(rng.choice([0, 1, 3, 6, 50], K + 1)))  # per-group (TTL mode only)
        ttl = np.array(rows, np.uint32)
        for c1 in range(4):
            for c2 in range(3):
                for c3 in range(4):
                    for ti in range(6):
                        caps.append([c1, c2, c3]); tuners.append(ti)
                for ti in range(1, len(rows)):
                    caps.append([c1, c2, INF]); tuners.append(ti)
        cf = O.configs(caps, tuner=np.array(tuners))
        got = ot.stack_counts(cf, ttl)
        want = ot.replay(cf, ttl)
        assert np.array_equal(got, want), trial


def test_non_eligible_configs_refused():
    ot = O.OracleTrace(ki.from_chains([[1, 2], [1, 3]], [0, 1]), top_k=1)
    ttl = np.array([[5, 7]], np.uint32)
    assert not ot.stack_eligible(O.configs([[1, 1, 1]]), ttl)            # per-group tau, finite disk
    assert ot.stack_eligible(O.configs([[1, 1, INF]]), ttl)              # TTL mode: eligible
    assert not ot.stack_eligible(O.configs([[1, 1, 1]], policy=O.FIFO))  # FIFO never
    with pytest.raises(O.OracleError):
        ot.stack_counts(O.configs([[1, 1, 1]]), ttl)

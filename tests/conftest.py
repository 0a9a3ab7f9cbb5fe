import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-size) test")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def chains_from_labels(chains, arrivals, hashes_of_root=None):
    """Sorted brute-force input from label chains: (arrival, group placeholder, block ids),
    block identity = label prefix tuple.  Stable sort by (arrival, file index)."""
    order = sorted(range(len(chains)), key=lambda i: (arrivals[i], i))
    out = []
    for i in order:
        ch = chains[i]
        out.append((int(arrivals[i]), 0, [tuple(ch[:k + 1]) for k in range(len(ch))]))
    return out


def assign_groups(sorted_chains, K, root_hash):
    """Top-K prefix-subtree groups: rank roots by (reuse desc, root hash asc)."""
    seen = set()
    reuse = {}
    for (_a, _g, ch) in sorted_chains:
        if not ch:
            continue
        rt = ch[0]
        reuse.setdefault(rt, 0)
        for b in ch:
            if b in seen:
                reuse[rt] += 1
            seen.add(b)
    ranked = sorted(reuse, key=lambda rt: (-reuse[rt], root_hash[rt]))
    rank = {rt: i for i, rt in enumerate(ranked)}
    out = []
    for (a, _g, ch) in sorted_chains:
        g = K if not ch else min(rank[ch[0]], K)
        out.append((a, g, ch))
    return out

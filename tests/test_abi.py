"""CPU checks of the C-ABI boundary: libkareto.so builds for sm_100a, loads, exports every
function include/kareto.h declares, struct layouts match, host-only helpers work.
No compute calls (there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2603_08739_b200 as K
from paper_2603_08739_b200 import build as kbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kareto.h")


@pytest.fixture(scope="module")
def lib():
    kbuild.build()
    return K.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kareto_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(K.ABI_FUNCTIONS) == names


def test_library_is_sm100a_only():
    kbuild.build()
    out = subprocess.run(["cuobjdump", "--list-elf", K.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_struct_layouts_match_header(lib):
    assert K.CONFIG_DTYPE.itemsize == 40
    assert K.COUNTS_DTYPE.itemsize == 88
    assert ctypes.sizeof(K.ModelC) == 4 * 2 + 8 * 4 + 8 * 6 + 4 * 2 + 32 * 8 + 24 * 8
    assert ctypes.sizeof(K.TraceDesc) == 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8  # 80 with padding


def test_shard_range_partitions(lib):
    for n in (0, 1, 7, 16384, 103680):
        for world in (1, 2, 3, 4, 8):
            parts = [K.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_time_slices_and_hash_owner(lib):
    """Host rules of the time-sharded load (kareto_time_slices, kareto_hash_owner): slices tile
    the sorted requests in order, each rank's first block position is the first request start at
    or after k N / W (requests without blocks included), owners cover [0, W) near-uniformly."""
    rng = np.random.default_rng(0)
    nb = rng.integers(0, 50, size=2000)
    nb[rng.integers(0, 2000, size=200)] = 0  # requests without full blocks
    s = np.concatenate([[0], np.cumsum(nb)]).astype(np.uint32)
    N = int(s[-1])
    for world in (1, 2, 3, 7, 8, 128):
        rb = K.time_slices(s, world)
        assert rb[0] == 0 and rb[-1] == len(s) - 1 and np.all(np.diff(rb) >= 0)
        for k in range(world):
            want = int(np.searchsorted(s[:-1], N * k // world, side="left"))
            assert rb[k] == want
    with pytest.raises(K.KaretoError):
        K.time_slices(s, 0)
    hs = rng.integers(0, 2**63, size=20000, dtype=np.int64).astype(np.uint64)
    for world in (1, 3, 8):
        own = np.array([K.hash_owner(int(h), world) for h in hs])
        assert own.min() >= 0 and own.max() < world
        cnt = np.bincount(own, minlength=world)
        assert cnt.min() > 0.8 * len(hs) / world
    assert K.hash_owner(123, 0) == -1


def test_invalid_arguments_without_gpu(lib):
    h = ctypes.c_void_p()
    assert lib.kareto_create(0, None, None, 2, 1, ctypes.byref(h)) == K.E_INVALID  # rank >= world
    assert lib.kareto_create(0, None, None, 0, 2, ctypes.byref(h)) == K.E_INVALID  # world > 1 without id
    with pytest.raises(K.KaretoError):
        K.shard_range(5, 3, 2)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2603_08739_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "kareto_oracle", "or_replay", "or_trace"):
                    assert bad not in txt, (f, bad)


def test_shard_bounds_cost_weighted():
    """kareto_shard_bounds (host-only): unit weights reproduce kareto_shard_range; replay
    configurations (FIFO here) weigh 10^6 stack configurations, so they are spread evenly."""
    import numpy as np
    import paper_2603_08739_b200 as K
    for n in (0, 1, 7, 100, 1001):
        cf = K.configs([[1, 2, 3]] * n)
        for world in (1, 2, 3, 8):
            b = K.shard_bounds(cf, world)
            assert [tuple(b[r:r + 2]) for r in range(world)] == [K.shard_range(n, r, world) for r in range(world)]
    pol = np.array([K.LRU] * 900 + [K.FIFO] * 100)
    cf = K.configs([[1, 2, 3]] * 1000, policy=pol)
    for world in (2, 4, 8):
        b = K.shard_bounds(cf, world)
        per = [int((pol[b[r]:b[r + 1]] == K.FIFO).sum()) for r in range(world)]
        assert max(per) - min(per) <= 2 and sum(per) == 100

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

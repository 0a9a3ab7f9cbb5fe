"""Seeded synthetic trace generators shared by the oracle tests and the CUDA path.

This package holds NONE of the method's arithmetic (no hashing, replay or cost
model).  It produces request arrays in the layout both implementations accept:

    arrival_ms   int64[R]   request arrival, ms (file order, not sorted)
    output_tokens int32[R]  decode length
    offsets      int64[R+1] token offsets of each request's input
    tokens       uint32[T]  input token ids

Large traces (G-chat / G-api / G-agent shaped like the
paper's traces A/B/C, PAPER.md 3.3 lines 368-374, 5 line 802) come from the
C generator in gen.c; tiny hand-built and random prefix-tree traces used by the
unit tests are built here in numpy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libkgen.so")
_lib = None

KINDS = {"chat": 0, "api": 1, "agent": 2}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", _SO, src, "-lm", "-lpthread"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.kg_plan_create.restype = ctypes.c_void_p
        lib.kg_plan_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64]
        for fn in ("kg_plan_requests", "kg_plan_tokens", "kg_plan_blocks"):
            getattr(lib, fn).restype = ctypes.c_int64
            getattr(lib, fn).argtypes = [ctypes.c_void_p]
        lib.kg_plan_fill_meta.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 3
        lib.kg_plan_fill_tokens.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.kg_plan_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclass
class Trace:
    """A request trace in file order (the library stable-sorts by arrival)."""

    arrival_ms: np.ndarray
    output_tokens: np.ndarray
    offsets: np.ndarray
    tokens: np.ndarray | None = None          # TOKENS mode
    block_hash: np.ndarray | None = None      # HASHES mode (offsets are block offsets)
    input_tokens: np.ndarray | None = None    # HASHES mode (optional)
    meta: dict = field(default_factory=dict)

    @property
    def n_requests(self) -> int:
        return int(self.arrival_ms.shape[0])

    @property
    def n_blocks(self) -> int:
        if self.tokens is not None:
            lens = np.diff(self.offsets)
            return int((lens // 16).sum())
        return int(self.offsets[-1])


class Plan:
    """A generated synthetic trace plan; arrays are filled on demand (large traces)."""

    def __init__(self, kind: str, R: int = 0, N: int = 0, seed: int = 0):
        lib = _load()
        self._lib = lib
        self._p = lib.kg_plan_create(KINDS[kind], int(R), int(N), int(seed))
        self.kind, self.seed = kind, seed
        self.n_requests = lib.kg_plan_requests(self._p)
        self.n_tokens = lib.kg_plan_tokens(self._p)
        self.n_blocks = lib.kg_plan_blocks(self._p)

    def fill_meta(self, arrival_ms: np.ndarray, output_tokens: np.ndarray, offsets: np.ndarray) -> None:
        assert arrival_ms.dtype == np.int64 and output_tokens.dtype == np.int32 and offsets.dtype == np.int64
        self._lib.kg_plan_fill_meta(self._p, arrival_ms.ctypes.data, output_tokens.ctypes.data, offsets.ctypes.data)

    def fill_tokens_ptr(self, ptr: int, threads: int | None = None) -> None:
        self._lib.kg_plan_fill_tokens(self._p, ctypes.c_void_p(ptr), int(threads or os.cpu_count() or 1))

    def materialize(self, threads: int | None = None) -> Trace:
        R = self.n_requests
        arr = np.empty(R, np.int64)
        out = np.empty(R, np.int32)
        off = np.empty(R + 1, np.int64)
        self.fill_meta(arr, out, off)
        tok = np.empty(self.n_tokens, np.uint32)
        self.fill_tokens_ptr(tok.ctypes.data, threads)
        return Trace(arr, out, off, tokens=tok, meta={"kind": self.kind, "seed": self.seed})

    def __del__(self):
        try:
            self._lib.kg_plan_free(self._p)
        except Exception:
            pass


def synthetic(kind: str = "chat", R: int = 0, N: int = 0, seed: int = 0, threads: int | None = None) -> Trace:
    return Plan(kind, R=R, N=N, seed=seed).materialize(threads)


# ----------------------------------------------------------------------------------
# tiny traces for unit tests
# ----------------------------------------------------------------------------------
def _block_tokens(label: int) -> np.ndarray:
    """16 token ids for a block label (labels are arbitrary non-negative ints)."""
    base = (label * 7919 + 13) % 1000003
    return (np.arange(16, dtype=np.uint32) * np.uint32(31) + np.uint32(base)).astype(np.uint32)


def from_chains(chains, arrivals, output_tokens=None, tails=None) -> Trace:
    """Build a TOKENS-mode trace whose request r consists of the blocks with the given
    labels (chains[r] = [label_0, label_1, ...]) followed by `tails[r]` extra tokens
    (< 16, a partial block that is never hashed).  Two requests share block k iff
    their label prefixes [0..k] are equal -- labels are just token patterns, the
    prefix identity comes from the chained hash."""
    R = len(chains)
    toks = []
    offs = [0]
    for r, ch in enumerate(chains):
        parts = [_block_tokens(int(x)) for x in ch]
        t = tails[r] if tails is not None else 0
        if t:
            parts.append(np.full(t, 7, np.uint32))
        seq = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
        toks.append(seq)
        offs.append(offs[-1] + len(seq))
    tokens = np.concatenate(toks) if toks else np.zeros(0, np.uint32)
    out = np.asarray(output_tokens if output_tokens is not None else [1] * R, np.int32)
    return Trace(np.asarray(arrivals, np.int64), out, np.asarray(offs, np.int64), tokens=tokens.astype(np.uint32))


def random_prefix_tree(rng: np.random.Generator, n_req: int = None, max_depth: int = 6,
                       fanout: int = 3, n_roots: int = 3, partial_tail: bool = True) -> Trace:
    """Random chain-consistent trace (SURVEY Appendix A generator): requests pick a
    root->node path in a random prefix tree; arrival increments from {0,0,1,2,3,5,8} ms."""
    if n_req is None:
        n_req = int(rng.integers(5, 41))
    chains = []
    for _ in range(n_req):
        depth = int(rng.integers(1, max_depth + 1))
        root = int(rng.integers(0, n_roots))
        ch = [root]
        for _d in range(depth - 1):
            ch.append(int(rng.integers(0, fanout)) + 100 * (len(ch)))
        chains.append(ch)
    inc = np.array([0, 0, 1, 2, 3, 5, 8])
    arr = np.cumsum(inc[rng.integers(0, len(inc), n_req)])
    tails = rng.integers(0, 16, n_req) if partial_tail else None
    outs = rng.integers(1, 50, n_req)
    # shuffle file order so the library's stable sort by arrival is exercised
    perm = rng.permutation(n_req)
    chains = [chains[i] for i in perm]
    arr = arr[perm]
    tails = tails[perm] if tails is not None else None
    outs = outs[perm]
    return from_chains(chains, arr, outs, tails)

"""ctypes wrapper of the C oracle (oracle/kareto_oracle.c).

TEST INFRASTRUCTURE ONLY: may be imported solely by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs.  The product package
paper_2603_08739_b200 never imports this module.

Configurations are passed in a neutral numpy form (see `configs()`), so this wrapper
shares no struct definition with the product's binding.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, E_INVALID, E_PARSE, E_CHAIN, E_OOM, E_OVERFLOW = 0, 1, 2, 3, 4, 7
LRU, FIFO, LFU = 0, 1, 2
INF_CAP = np.uint64(0xFFFFFFFFFFFFFFFF)
INF_TTL = np.uint32(0xFFFFFFFF)
NA = 0xFFFFFFFFFFFFFFFF


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "kareto_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                               "-o", _SO, src, "-lpthread"])
    return _SO


class _Desc(ctypes.Structure):
    _fields_ = [("n_requests", ctypes.c_int64), ("arrival_ms", ctypes.c_void_p), ("output_tokens", ctypes.c_void_p),
                ("mode", ctypes.c_int32), ("offsets", ctypes.c_void_p), ("tokens", ctypes.c_void_p),
                ("block_hash", ctypes.c_void_p), ("input_tokens", ctypes.c_void_p), ("salt", ctypes.c_uint64),
                ("top_k", ctypes.c_int32)]


# neutral config layout used by the tests; the oracle's C struct happens to be 40 bytes
CONFIG_DTYPE = np.dtype([("cap", "<u8", (3,)), ("policy", "u1"), ("medium", "u1"), ("tuner", "<u2"),
                         ("axis", "<i4", (3,))], align=True)
COUNTS_DTYPE = np.dtype([("hit", "<u8", (3,)), ("miss", "<u8"), ("evict", "<u8", (3,)), ("disk_writes", "<u8"),
                         ("hit_pos_sum", "<u8"), ("bytetime_block_ms", "<u8"), ("resident_after_hole", "<u8")])
COUNT_FIELDS = ["hit", "miss", "evict", "disk_writes", "hit_pos_sum", "bytetime_block_ms", "resident_after_hole"]


class _Medium(ctypes.Structure):
    _fields_ = [("bw_base", ctypes.c_double), ("bw_slope", ctypes.c_double), ("bw_max", ctypes.c_double),
                ("price", ctypes.c_double)]


class _Phi(ctypes.Structure):
    _fields_ = [("breakpoint", ctypes.c_double), ("rate", ctypes.c_double), ("jump", ctypes.c_double)]


class _Model(ctypes.Structure):
    _fields_ = [("instances", ctypes.c_int32), ("gpus_per_instance", ctypes.c_int32),
                ("alpha_ps", ctypes.c_uint64), ("beta_ps", ctypes.c_uint64), ("dec_ps", ctypes.c_uint64),
                ("block_bytes", ctypes.c_uint64), ("bw_dram", ctypes.c_double), ("c_hw", ctypes.c_double),
                ("p_hbm", ctypes.c_double), ("p_dram", ctypes.c_double), ("iops_per_block", ctypes.c_double),
                ("ttl_prov_gb", ctypes.c_double), ("n_media", ctypes.c_int32), ("n_phi", ctypes.c_int32),
                ("media", _Medium * 8), ("phi", _Phi * 8)]


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(_SO)
    vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
    L.or_trace_build.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(vp)]
    L.or_trace_free.argtypes = [vp]
    L.or_trace_stats.argtypes = [vp] + [vp] * 8
    L.or_trace_export.argtypes = [vp] + [vp] * 7
    L.or_replay_many.argtypes = [vp, vp, i64, vp, i32, vp, ctypes.c_int]
    L.or_replay_lookup.argtypes = [vp, vp, vp, vp, vp]
    L.or_stack_create.restype = vp
    L.or_stack_create.argtypes = [vp]
    L.or_stack_free.argtypes = [vp]
    L.or_stack_export.argtypes = [vp, vp, vp]
    L.or_stack_counts.argtypes = [vp, vp, vp, vp]
    L.or_stack_eligible.argtypes = [vp, vp, vp]
    L.or_objective_many.argtypes = [vp, ctypes.POINTER(_Model), vp, vp, i64, vp]
    L.or_prune.argtypes = [vp, vp, i64, ctypes.c_double, vp]
    L.or_pareto.restype = i64
    L.or_pareto.argtypes = [vp, i64, vp, vp]
    L.or_objective_many_mt.argtypes = [vp, vp, vp, vp, i64, vp, ctypes.c_int]
    L.or_pareto_mt.restype = i64
    L.or_pareto_mt.argtypes = [vp, i64, vp, vp, ctypes.c_int]
    L.or_fmix64_export.restype = u64
    L.or_fmix64_export.argtypes = [u64]
    L.or_content_hash_export.restype = u64
    L.or_content_hash_export.argtypes = [vp]
    L.or_chain_hashes.argtypes = [vp, i64, u64, vp]
    L.or_phi.restype = ctypes.c_double
    L.or_phi.argtypes = [ctypes.POINTER(_Model), ctypes.c_double]
    L.or_prefill_p0.argtypes = [vp, ctypes.POINTER(_Model), vp]
    _lib = L
    return L


def _ptr(a):
    return None if a is None else a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"oracle status {status} {what}")
        self.status = status


def fmix64(x: int) -> int:
    return int(_load().or_fmix64_export(ctypes.c_uint64(x)))


def content_hash(tokens16) -> int:
    t = np.ascontiguousarray(tokens16, np.uint32)
    assert t.shape == (16,)
    return int(_load().or_content_hash_export(t.ctypes.data))


def chain_hashes(tokens, salt: int = 0) -> np.ndarray:
    t = np.ascontiguousarray(tokens, np.uint32)
    out = np.zeros(len(t) // 16, np.uint64)
    _load().or_chain_hashes(t.ctypes.data, len(t), ctypes.c_uint64(salt), out.ctypes.data)
    return out


def configs(caps, policy=0, medium=0, tuner=0, axis=None) -> np.ndarray:
    """Neutral config array: caps [n,3] uint64 (INF_CAP allowed for cap[2])."""
    caps = np.asarray(caps, dtype=np.uint64).reshape(-1, 3)
    n = caps.shape[0]
    c = np.zeros(n, CONFIG_DTYPE)
    c["cap"] = caps
    c["policy"] = policy
    c["medium"] = medium
    c["tuner"] = tuner
    if axis is not None:
        c["axis"] = np.asarray(axis, np.int32).reshape(n, 3)
    return c


class Model:
    """Objective-model constants; defaults = SURVEY 8.d.3 bench constants."""

    def __init__(self, instances=1, gpus_per_instance=8, alpha_ps=50_000_000, beta_ps=1, dec_ps=150_000_000,
                 block_bytes=5_242_880, bw_dram=25e9, c_hw=2.5, p_hbm=0.0, p_dram=0.004, iops_per_block=1.0,
                 ttl_prov_gb=1024.0, media=((120e6, 0.5e6, 350e6, 0.0001),),
                 phi=((0.0, 0.0, 0.0), (3000.0, 0.005, 0.0), (32000.0, 0.065, 0.0))):
        self.__dict__.update(dict(instances=instances, gpus_per_instance=gpus_per_instance, alpha_ps=alpha_ps,
                                  beta_ps=beta_ps, dec_ps=dec_ps, block_bytes=block_bytes, bw_dram=bw_dram,
                                  c_hw=c_hw, p_hbm=p_hbm, p_dram=p_dram, iops_per_block=iops_per_block,
                                  ttl_prov_gb=ttl_prov_gb, media=tuple(media), phi=tuple(phi)))

    def _c(self) -> _Model:
        m = _Model()
        for k in ("instances", "gpus_per_instance", "alpha_ps", "beta_ps", "dec_ps", "block_bytes", "bw_dram",
                  "c_hw", "p_hbm", "p_dram", "iops_per_block", "ttl_prov_gb"):
            setattr(m, k, getattr(self, k))
        m.n_media = len(self.media)
        for i, (a, b, c, d) in enumerate(self.media):
            m.media[i].bw_base, m.media[i].bw_slope, m.media[i].bw_max, m.media[i].price = a, b, c, d
        m.n_phi = len(self.phi)
        for i, (a, b, c) in enumerate(self.phi):
            m.phi[i].breakpoint, m.phi[i].rate, m.phi[i].jump = a, b, c
        return m


def phi(model: Model, u: float) -> float:
    m = model._c()
    return float(_load().or_phi(ctypes.byref(m), ctypes.c_double(u)))


class OracleTrace:
    """Oracle trace: O-1..O-6 of DESIGN.md "Oracle" (sort, hash, prev/delta, chain check, groups)."""

    def __init__(self, trace, salt: int = 0, top_k: int = 16, mode: str | None = None):
        L = _load()
        self._L = L
        mode = mode or ("tokens" if trace.tokens is not None else "hashes")
        self._keep = []
        d = _Desc()
        d.n_requests = trace.n_requests
        arr = np.ascontiguousarray(trace.arrival_ms, np.int64)
        out = np.ascontiguousarray(trace.output_tokens, np.int32)
        off = np.ascontiguousarray(trace.offsets, np.int64)
        self._keep += [arr, out, off]
        d.arrival_ms, d.output_tokens, d.offsets = arr.ctypes.data, out.ctypes.data, off.ctypes.data
        if mode == "tokens":
            tok = np.ascontiguousarray(trace.tokens, np.uint32)
            self._keep.append(tok)
            d.mode, d.tokens = 0, tok.ctypes.data if tok.size else None
        else:
            bh = np.ascontiguousarray(trace.block_hash, np.uint64)
            self._keep.append(bh)
            d.mode, d.block_hash = 1, bh.ctypes.data if bh.size else None
            if trace.input_tokens is not None:
                it = np.ascontiguousarray(trace.input_tokens, np.int64)
                self._keep.append(it)
                d.input_tokens = it.ctypes.data
        d.salt = salt
        d.top_k = top_k
        h = ctypes.c_void_p()
        st = L.or_trace_build(ctypes.byref(d), ctypes.byref(h))
        if st != OK:
            raise OracleError(st, "trace_build")
        self._h = h
        self.K = top_k
        self._stack = None
        v = [ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_uint64(),
             ctypes.c_uint64()]
        self.U_g = np.zeros(top_k + 1, np.int64)
        self.reuse_g = np.zeros(top_k + 1, np.int64)
        L.or_trace_stats(h, *[ctypes.addressof(x) for x in v], self.U_g.ctypes.data, self.reuse_g.ctypes.data)
        self.R, self.N, self.U, self.span_ms, self.Ltok, self.O = [int(x.value) for x in v]

    def __del__(self):
        try:
            if self._stack is not None:
                self._L.or_stack_free(self._stack)
            self._L.or_trace_free(self._h)
        except Exception:
            pass

    def export(self) -> dict:
        N, R = self.N, self.R
        e = dict(hash=np.zeros(N, np.uint64), prev=np.zeros(N, np.int64), delta=np.zeros(N, np.int64),
                 req=np.zeros(N, np.int32), k=np.zeros(N, np.int32), group=np.zeros(R, np.int32),
                 s=np.zeros(R + 1, np.int64))
        self._L.or_trace_export(self._h, e["hash"].ctypes.data, e["prev"].ctypes.data, e["delta"].ctypes.data,
                                e["req"].ctypes.data, e["k"].ctypes.data, e["group"].ctypes.data,
                                e["s"].ctypes.data)
        return e

    # ---- O1 --------------------------------------------------------------------
    def replay(self, cfgs: np.ndarray, ttl=None, threads: int | None = None) -> np.ndarray:
        ttl = self._ttl(ttl)
        cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        out = np.zeros(len(cfgs), COUNTS_DTYPE)
        st = self._L.or_replay_many(self._h, cfgs.ctypes.data, len(cfgs), ttl.ctypes.data, ttl.shape[0],
                                    out.ctypes.data, int(threads or os.cpu_count() or 1))
        if st != OK:
            raise OracleError(st, "replay")
        return out

    def replay_lookup(self, cfg, ttl=None):
        """O1 for one configuration plus, per access (touch order), the tier that served it in
        its request's hit prefix (1 HBM, 2 DRAM, 3 disk / lease), 0 outside (row f3)."""
        ttl = self._ttl(ttl)
        c = np.ascontiguousarray(np.atleast_1d(cfg)[:1], CONFIG_DTYPE)
        row = np.ascontiguousarray(ttl[int(c[0]["tuner"])])
        out = np.zeros(1, COUNTS_DTYPE)
        lt = np.zeros(max(self.N, 1), np.uint8)
        st = self._L.or_replay_lookup(self._h, c.ctypes.data, row.ctypes.data, out.ctypes.data, lt.ctypes.data)
        if st != OK:
            raise OracleError(st, "replay_lookup")
        return out[0], lt[:self.N]

    def _ttl(self, ttl):
        if ttl is None:
            ttl = np.full((1, self.K + 1), INF_TTL, np.uint32)
        ttl = np.ascontiguousarray(ttl, np.uint32)
        assert ttl.ndim == 2 and ttl.shape[1] == self.K + 1
        return ttl

    # ---- O2 --------------------------------------------------------------------
    def _stk(self):
        if self._stack is None:
            self._stack = self._L.or_stack_create(self._h)
        return self._stack

    def depth(self):
        d = np.zeros(self.N, np.int64)
        D = np.zeros(self.N, np.int64)
        self._L.or_stack_export(self._stk(), d.ctypes.data, D.ctypes.data)
        return d, D

    def stack_eligible(self, cfg, ttl=None) -> bool:
        ttl = self._ttl(ttl)
        c = np.ascontiguousarray(np.atleast_1d(cfg), CONFIG_DTYPE)
        row = np.ascontiguousarray(ttl[int(c[0]["tuner"])])
        return bool(self._L.or_stack_eligible(self._h, c.ctypes.data, row.ctypes.data))

    def stack_counts(self, cfgs: np.ndarray, ttl=None) -> np.ndarray:
        ttl = self._ttl(ttl)
        cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        out = np.zeros(len(cfgs), COUNTS_DTYPE)
        stk = self._stk()
        for i in range(len(cfgs)):
            row = np.ascontiguousarray(ttl[int(cfgs[i]["tuner"])])
            st = self._L.or_stack_counts(stk, cfgs[i:i + 1].ctypes.data, row.ctypes.data, out[i:i + 1].ctypes.data)
            if st != OK:
                raise OracleError(st, f"stack_counts[{i}]")
        return out

    # ---- model / selection -----------------------------------------------------------
    def objective(self, model: Model, cfgs: np.ndarray, counts: np.ndarray, threads: int = 1) -> np.ndarray:
        """fp64 objectives (R25-R33); threads > 1 splits the configurations across host threads."""
        cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        counts = np.ascontiguousarray(counts, COUNTS_DTYPE)
        f = np.zeros((len(cfgs), 3), np.float64)
        m = model._c()
        if threads > 1:
            st = self._L.or_objective_many_mt(self._h, ctypes.byref(m), cfgs.ctypes.data, counts.ctypes.data,
                                              len(cfgs), f.ctypes.data, int(threads))
        else:
            st = self._L.or_objective_many(self._h, ctypes.byref(m), cfgs.ctypes.data, counts.ctypes.data,
                                           len(cfgs), f.ctypes.data)
        if st != OK:
            raise OracleError(st, "objective")
        return f

    def prefill_p0(self, model: Model) -> int:
        v = ctypes.c_uint64()
        m = model._c()
        st = self._L.or_prefill_p0(self._h, ctypes.byref(m), ctypes.addressof(v))
        if st != OK:
            raise OracleError(st, "p0")
        return int(v.value)


def prune(f: np.ndarray, cfgs: np.ndarray, tau_e: float = 0.05) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float64)
    cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
    out = np.zeros(len(cfgs), np.uint8)
    _load().or_prune(f.ctypes.data, cfgs.ctypes.data, len(cfgs), ctypes.c_double(tau_e), out.ctypes.data)
    return out


def pareto(f: np.ndarray, pruned: np.ndarray | None = None, threads: int = 1) -> np.ndarray:
    """O(n^2) dominance (R35); threads > 1 splits the rows across host threads (same result)."""
    f = np.ascontiguousarray(f, np.float64)
    n = f.shape[0]
    st = np.zeros(n, np.uint8)
    pr = None if pruned is None else np.ascontiguousarray(pruned, np.uint8)
    if threads > 1:
        _load().or_pareto_mt(f.ctypes.data, n, _ptr(pr), st.ctypes.data, int(threads))
    else:
        _load().or_pareto(f.ctypes.data, n, _ptr(pr), st.ctypes.data)
    return st


def select(f, cfgs, tau_e: float | None = 0.05, threads: int = 1) -> np.ndarray:
    """Full kareto_pareto semantics: status 2 pruned / 1 frontier / 0 dominated."""
    pr = prune(f, cfgs, tau_e) if tau_e is not None else None
    return pareto(f, pr, threads)


def timed_replay(tr: OracleTrace, cfgs, ttl=None, threads=None):
    t0 = time.perf_counter()
    c = tr.replay(cfgs, ttl, threads)
    return c, time.perf_counter() - t0

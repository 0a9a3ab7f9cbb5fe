"""kareto-b200: B200-native hot path of Kareto's configuration search (arXiv 2603.08739).

Thin ctypes binding of the C ABI in include/kareto.h (libkareto.so, built in-tree by
paper_2603_08739_b200.build).  Argument marshalling only: every step of the path runs in
the library's CUDA kernels.  There is no CPU fallback -- importing works without a GPU
(for the ABI export checks) but every compute call needs the CUDA library and a device.

Names follow the ABI: load_trace / eval_grid / pareto.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkareto.so")

OK, E_INVALID, E_PARSE, E_CHAIN, E_OOM, E_CUDA, E_NCCL, E_OVERFLOW, E_UNSUPPORTED = range(9)
STATUS_NAMES = ["OK", "E_INVALID", "E_PARSE", "E_CHAIN", "E_OOM", "E_CUDA", "E_NCCL", "E_OVERFLOW", "E_UNSUPPORTED"]
TOKENS, HASHES = 0, 1
LRU, FIFO, LFU = 0, 1, 2
INF = 0xFFFFFFFFFFFFFFFF
NA = 0xFFFFFFFFFFFFFFFF
TTL_INF = 0xFFFFFFFF
X_HASH, X_PREV, X_DELTA, X_REQ, X_DEPTH, X_GROUP, X_START = range(7)

# struct layouts of include/kareto.h
CONFIG_DTYPE = np.dtype([("cap", "<u8", (3,)), ("policy", "u1"), ("medium", "u1"), ("tuner", "<u2"),
                         ("axis", "<i4", (3,))], align=True)
COUNTS_DTYPE = np.dtype([("hit", "<u8", (3,)), ("miss", "<u8"), ("evict", "<u8", (3,)), ("disk_writes", "<u8"),
                         ("hit_pos_sum", "<u8"), ("bytetime_block_ms", "<u8"), ("resident_after_hole", "<u8")])
assert CONFIG_DTYPE.itemsize == 40 and COUNTS_DTYPE.itemsize == 88


class KaretoError(RuntimeError):
    def __init__(self, status: int, message: str = ""):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"kareto {name}: {message}")
        self.status = status


class TraceDesc(ctypes.Structure):
    _fields_ = [("n_requests", ctypes.c_int64), ("arrival_ms", ctypes.c_void_p), ("output_tokens", ctypes.c_void_p),
                ("mode", ctypes.c_int32), ("offsets", ctypes.c_void_p), ("tokens", ctypes.c_void_p),
                ("block_hash", ctypes.c_void_p), ("input_tokens", ctypes.c_void_p), ("salt", ctypes.c_uint64),
                ("top_k", ctypes.c_int32), ("inputs_on_device", ctypes.c_int32)]


class TraceInfo(ctypes.Structure):
    _fields_ = [("n_requests", ctypes.c_int64), ("n_accesses", ctypes.c_int64), ("n_unique", ctypes.c_int64),
                ("span_ms", ctypes.c_int64), ("input_tokens", ctypes.c_uint64), ("output_tokens", ctypes.c_uint64),
                ("top_k", ctypes.c_int32), ("max_blocks_per_request", ctypes.c_int32)]


class Medium(ctypes.Structure):
    _fields_ = [("bw_base", ctypes.c_double), ("bw_slope", ctypes.c_double), ("bw_max", ctypes.c_double),
                ("price", ctypes.c_double)]


class PhiSegment(ctypes.Structure):
    _fields_ = [("breakpoint", ctypes.c_double), ("rate", ctypes.c_double), ("jump", ctypes.c_double)]


class ModelC(ctypes.Structure):
    _fields_ = [("instances", ctypes.c_int32), ("gpus_per_instance", ctypes.c_int32), ("alpha_ps", ctypes.c_uint64),
                ("beta_ps", ctypes.c_uint64), ("dec_ps", ctypes.c_uint64), ("block_bytes", ctypes.c_uint64),
                ("bw_dram", ctypes.c_double), ("c_hw", ctypes.c_double), ("p_hbm", ctypes.c_double),
                ("p_dram", ctypes.c_double), ("iops_per_block", ctypes.c_double), ("ttl_prov_gb", ctypes.c_double),
                ("n_media", ctypes.c_int32), ("n_phi", ctypes.c_int32), ("media", Medium * 8), ("phi", PhiSegment * 8)]


class PruneC(ctypes.Structure):
    _fields_ = [("enabled", ctypes.c_int32), ("tau_e", ctypes.c_double)]


class SearchParamsC(ctypes.Structure):
    _fields_ = [("hbm_gb", ctypes.c_double), ("d_min", ctypes.c_int64), ("d_max", ctypes.c_int64),
                ("d_step", ctypes.c_int64), ("t_min", ctypes.c_int64), ("t_max", ctypes.c_int64),
                ("t_step", ctypes.c_int64), ("tau_e", ctypes.c_double), ("tau_perf", ctypes.c_double),
                ("tau_cost", ctypes.c_double), ("policy", ctypes.c_int32), ("max_rounds", ctypes.c_int32),
                ("expand_ttl", ctypes.c_int32), ("pad", ctypes.c_int32)]


# kareto_search_point (48 bytes)
SEARCH_POINT_DTYPE = np.dtype([("d_gb", np.int64), ("t_s", np.int64), ("obj", np.float64, 3), ("round", np.int32),
                               ("status", np.uint8), ("pad", np.uint8, 3)])
assert SEARCH_POINT_DTYPE.itemsize == 48


class AnalyticsC(ctypes.Structure):
    _fields_ = [("unique_blocks", ctypes.c_int64), ("total_hits", ctypes.c_int64), ("blocks_90", ctypes.c_int64),
                ("frac_90", ctypes.c_double), ("peak_active", ctypes.c_int64),
                ("peak_active_request", ctypes.c_int64), ("final_cumulative", ctypes.c_int64)]


# kareto_queue_result (48 bytes)
QUEUE_DTYPE = np.dtype([("ttft_mean_ms", np.float64), ("ttft_p99_ms", np.float64), ("makespan_s", np.float64),
                        ("tokens_per_s", np.float64), ("disk_hits_capacity", np.uint64),
                        ("disk_hits_realized", np.uint64)])
assert QUEUE_DTYPE.itemsize == 48


class PassTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("ms", ctypes.c_double), ("launches", ctypes.c_int32),
                ("own", ctypes.c_int32)]


_lib = None

# every function declared in include/kareto.h (checked by tests/test_abi.py)
ABI_FUNCTIONS = ["kareto_create", "kareto_destroy", "kareto_last_error", "kareto_nccl_unique_id",
                 "kareto_load_trace", "kareto_trace_free", "kareto_trace_stats", "kareto_trace_export",
                 "kareto_eval_grid", "kareto_pareto", "kareto_set_profiling", "kareto_get_pass_times",
                 "kareto_launch_counter", "kareto_shard_range", "kareto_shard_bounds", "kareto_hypervolume", "kareto_search",
                 "kareto_ttl_roi", "kareto_ttl_eval", "kareto_ttl_allocate", "kareto_trace_analytics",
                 "kareto_eval_queue", "kareto_loopback_create", "kareto_loopback_destroy", "kareto_loopback_world",
                 "kareto_create_loopback", "kareto_load_trace_sharded", "kareto_trace_shard", "kareto_time_slices",
                 "kareto_hash_owner", "kareto_grid_create", "kareto_grid_free", "kareto_eval_grid_prepared",
                 "kareto_pareto_prepared"]


def load_library(path: str = LIB_PATH):
    """Load libkareto.so; raises if it is missing (there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libkareto.so not built ({path}); run `python -m paper_2603_08739_b200.build`")
    L = ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.kareto_create.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.kareto_destroy.argtypes = [vp]
    L.kareto_destroy.restype = None
    L.kareto_last_error.argtypes = [vp]
    L.kareto_last_error.restype = ctypes.c_char_p
    L.kareto_nccl_unique_id.argtypes = [vp]
    L.kareto_load_trace.argtypes = [vp, ctypes.POINTER(TraceDesc), ctypes.POINTER(vp)]
    L.kareto_trace_free.argtypes = [vp]
    L.kareto_trace_free.restype = None
    L.kareto_trace_stats.argtypes = [vp, ctypes.POINTER(TraceInfo), vp, vp]
    L.kareto_trace_export.argtypes = [vp, vp, i32, vp]
    L.kareto_eval_grid.argtypes = [vp, vp, vp, i64, vp, i32, ctypes.POINTER(ModelC), vp, vp, i32]
    L.kareto_pareto.argtypes = [vp, vp, vp, i64, ctypes.POINTER(PruneC), vp, ctypes.POINTER(i64), i32]
    L.kareto_grid_create.argtypes = [vp, vp, i64, vp, i32, i32, ctypes.POINTER(vp)]
    L.kareto_grid_free.argtypes = [vp]
    L.kareto_grid_free.restype = None
    L.kareto_eval_grid_prepared.argtypes = [vp, vp, vp, ctypes.POINTER(ModelC), vp, vp, i32]
    L.kareto_pareto_prepared.argtypes = [vp, vp, vp, ctypes.POINTER(PruneC), vp, ctypes.POINTER(i64), i32]
    L.kareto_hypervolume.argtypes = [vp, vp, vp, i64, ctypes.POINTER(ctypes.c_double * 3),
                                     ctypes.POINTER(ctypes.c_double), i32]
    L.kareto_search.argtypes = [vp, vp, ctypes.POINTER(SearchParamsC), ctypes.POINTER(ModelC), vp, i64,
                                ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.kareto_ttl_roi.argtypes = [vp, vp, vp, vp, vp]
    L.kareto_ttl_eval.argtypes = [vp, vp, vp, i64, vp, vp]
    L.kareto_ttl_allocate.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_uint64, vp, ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.POINTER(ctypes.c_uint64), vp, vp]
    L.kareto_trace_analytics.argtypes = [vp, vp, ctypes.POINTER(AnalyticsC), vp, i32, vp, vp]
    L.kareto_eval_queue.argtypes = [vp, vp, vp, i64, vp, i32, ctypes.POINTER(ModelC), vp]
    L.kareto_set_profiling.argtypes = [vp, i32]
    L.kareto_get_pass_times.argtypes = [vp, ctypes.POINTER(PassTime), i32, ctypes.POINTER(i32), i32]
    L.kareto_launch_counter.argtypes = [vp, ctypes.POINTER(i64), i32]
    L.kareto_shard_range.argtypes = [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.kareto_shard_bounds.argtypes = [vp, i64, vp, i32, i32, i32, vp]
    L.kareto_loopback_create.argtypes = [i32, ctypes.POINTER(vp)]
    L.kareto_loopback_destroy.argtypes = [vp]
    L.kareto_loopback_destroy.restype = None
    L.kareto_loopback_world.argtypes = [vp]
    L.kareto_loopback_world.restype = i32
    L.kareto_create_loopback.argtypes = [ctypes.c_int, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    L.kareto_load_trace_sharded.argtypes = [vp, ctypes.POINTER(TraceDesc), ctypes.POINTER(vp)]
    L.kareto_time_slices.argtypes = [vp, i64, i32, vp]
    L.kareto_hash_owner.argtypes = [ctypes.c_uint64, i32]
    L.kareto_hash_owner.restype = i32
    L.kareto_trace_shard.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64),
                                     ctypes.POINTER(i64)]
    _lib = L
    return L


def _ptr(x):
    """(pointer, on_device) for a numpy array (host) or a torch tensor / CUDA-array-interface object."""
    if x is None:
        return None, False
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "arrays must be contiguous"
        return (x.ctypes.data if x.size else None), False
    if hasattr(x, "data_ptr"):
        return (x.data_ptr() or None), bool(getattr(x, "is_cuda", False))
    if hasattr(x, "__cuda_array_interface__"):
        return x.__cuda_array_interface__["data"][0], True
    raise TypeError(f"unsupported buffer {type(x)}")


def _check_outputs(counts, obj, n: int):
    """(counts ptr, obj ptr, on_device) after checking both live in one memory space with exactly
    88 * n / 24 * n contiguous bytes (float64 objectives)."""
    pc, dc = _ptr(counts)
    po, do = _ptr(obj)
    if counts is not None and obj is not None and dc != do:
        raise ValueError("counts and obj must both be host or both be device buffers")
    for name, buf, nbytes in (("counts", counts, 88 * n), ("obj", obj, 24 * n)):
        if buf is None:
            continue
        size = buf.nbytes if isinstance(buf, np.ndarray) else int(buf.numel()) * int(buf.element_size())
        if size != nbytes:
            raise ValueError(f"{name} must hold exactly {nbytes} bytes for {n} configurations, got {size}")
        if not isinstance(buf, np.ndarray) and not buf.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    if obj is not None and not isinstance(obj, np.ndarray) and "float64" not in str(obj.dtype):
        raise ValueError("obj must be float64 [n][3]")
    return pc, po, bool(dc or do)


class Model:
    """kareto_model constants; defaults = SURVEY 8.d.3 bench constants."""

    FIELDS = ("instances", "gpus_per_instance", "alpha_ps", "beta_ps", "dec_ps", "block_bytes", "bw_dram", "c_hw",
              "p_hbm", "p_dram", "iops_per_block", "ttl_prov_gb")

    def __init__(self, instances=1, gpus_per_instance=8, alpha_ps=50_000_000, beta_ps=1, dec_ps=150_000_000,
                 block_bytes=5_242_880, bw_dram=25e9, c_hw=2.5, p_hbm=0.0, p_dram=0.004, iops_per_block=1.0,
                 ttl_prov_gb=1024.0, media=((120e6, 0.5e6, 350e6, 0.0001),),
                 phi=((0.0, 0.0, 0.0), (3000.0, 0.005, 0.0), (32000.0, 0.065, 0.0))):
        self.instances, self.gpus_per_instance = instances, gpus_per_instance
        self.alpha_ps, self.beta_ps, self.dec_ps, self.block_bytes = alpha_ps, beta_ps, dec_ps, block_bytes
        self.bw_dram, self.c_hw, self.p_hbm, self.p_dram = bw_dram, c_hw, p_hbm, p_dram
        self.iops_per_block, self.ttl_prov_gb = iops_per_block, ttl_prov_gb
        self.media, self.phi = tuple(media), tuple(phi)

    def c(self) -> ModelC:
        m = ModelC()
        for k in self.FIELDS:
            setattr(m, k, getattr(self, k))
        m.n_media = len(self.media)
        for i, v in enumerate(self.media):
            m.media[i] = Medium(*v)
        m.n_phi = len(self.phi)
        for i, v in enumerate(self.phi):
            m.phi[i] = PhiSegment(*v)
        return m

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k in self.FIELDS}
        d["media"], d["phi"] = [list(x) for x in self.media], [list(x) for x in self.phi]
        return d


def configs(caps, policy=0, medium=0, tuner=0, axis=None) -> np.ndarray:
    """Build a kareto_config array from capacities [n,3] (uint64, INF allowed for cap[2])."""
    caps = np.asarray(caps, dtype=np.uint64).reshape(-1, 3)
    c = np.zeros(caps.shape[0], CONFIG_DTYPE)
    c["cap"] = caps
    c["policy"], c["medium"], c["tuner"] = policy, medium, tuner
    if axis is not None:
        c["axis"] = np.asarray(axis, np.int32).reshape(-1, 3)
    return c


class Loopback:
    """kareto_loopback: an in-process rank group (one host thread per rank, one device)."""

    def __init__(self, world: int):
        self._L = load_library()
        h = ctypes.c_void_p()
        st = self._L.kareto_loopback_create(world, ctypes.byref(h))
        if st != OK:
            raise KaretoError(st, "kareto_loopback_create")
        self._h, self.world = h, world

    def close(self):
        if getattr(self, "_h", None):
            self._L.kareto_loopback_destroy(self._h)
            self._h = None


class Context:
    """kareto_ctx: device, borrowed CUDA stream (an int handle, e.g. torch's
    current_stream().cuda_stream), optional NCCL communicator for world > 1, or a rank of a
    Loopback group (`loopback=`)."""

    def __init__(self, device: int = 0, stream: int | None = None, nccl_id: bytes | None = None, rank: int = 0,
                 world: int = 1, loopback: Loopback | None = None):
        self._L = load_library()
        h = ctypes.c_void_p()
        if loopback is not None:
            st = self._L.kareto_create_loopback(device, ctypes.c_void_p(stream or 0), loopback._h, rank,
                                                ctypes.byref(h))
            world = loopback.world
        else:
            nid = None
            if nccl_id is not None:
                nid = ctypes.create_string_buffer(bytes(nccl_id), 128)
            st = self._L.kareto_create(device, ctypes.c_void_p(stream or 0), nid, rank, world, ctypes.byref(h))
        if st != OK:
            raise KaretoError(st, "kareto_create")
        self._h = h
        self._loopback = loopback  # keep the group alive as long as the context
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        L = load_library()
        buf = ctypes.create_string_buffer(128)
        st = L.kareto_nccl_unique_id(buf)
        if st != OK:
            raise KaretoError(st, "kareto_nccl_unique_id")
        return buf.raw

    def _check(self, st: int, what: str):
        if st != OK:
            msg = self._L.kareto_last_error(self._h)
            raise KaretoError(st, f"{what}: {msg.decode(errors='replace') if msg else ''}")

    def close(self):
        if getattr(self, "_h", None):
            self._L.kareto_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- profiling --
    def set_profiling(self, on: bool = True):
        self._check(self._L.kareto_set_profiling(self._h, int(on)), "set_profiling")

    def pass_times(self, reset: bool = True) -> list[dict]:
        arr = (PassTime * 64)()
        n = ctypes.c_int32()
        self._check(self._L.kareto_get_pass_times(self._h, arr, 64, ctypes.byref(n), int(reset)), "pass_times")
        return [dict(name=arr[i].name.decode(), ms=arr[i].ms, launches=arr[i].launches, own=bool(arr[i].own))
                for i in range(n.value)]

    def launch_counter(self, reset: bool = False) -> int:
        v = ctypes.c_int64()
        self._check(self._L.kareto_launch_counter(self._h, ctypes.byref(v), int(reset)), "launch_counter")
        return int(v.value)

    # -------------------------------------------------------------------- ABI --
    def load_trace(self, arrival_ms, output_tokens, offsets, tokens=None, block_hash=None, input_tokens=None,
                   salt: int = 0, top_k: int = 16, time_shard: bool = False) -> "Trace":
        """kareto_load_trace (or, with time_shard, the collective kareto_load_trace_sharded).
        Arrays are all host numpy arrays or all device tensors."""
        d = TraceDesc()
        pa, dev = _ptr(arrival_ms)
        d.n_requests = int(arrival_ms.shape[0])
        d.arrival_ms = pa
        d.output_tokens = _ptr(output_tokens)[0]
        d.offsets = _ptr(offsets)[0]
        if tokens is not None:
            d.mode, d.tokens = TOKENS, _ptr(tokens)[0]
        else:
            d.mode, d.block_hash = HASHES, _ptr(block_hash)[0]
            d.input_tokens = _ptr(input_tokens)[0]
        d.salt, d.top_k, d.inputs_on_device = salt, top_k, int(dev)
        h = ctypes.c_void_p()
        fn = self._L.kareto_load_trace_sharded if time_shard else self._L.kareto_load_trace
        self._check(fn(self._h, ctypes.byref(d), ctypes.byref(h)), "load_trace")
        return Trace(self, h)

    def load(self, trace, salt: int = 0, top_k: int = 16, time_shard: bool = False) -> "Trace":
        """Load a kareto_inputs.Trace-like object (host arrays)."""
        return self.load_trace(trace.arrival_ms, trace.output_tokens, trace.offsets, tokens=trace.tokens,
                               block_hash=trace.block_hash, input_tokens=trace.input_tokens, salt=salt, top_k=top_k,
                               time_shard=time_shard)

    def eval_grid(self, trace: "Trace", cfgs: np.ndarray, model: Model, ttl=None, counts=None, obj=None):
        """kareto_eval_grid.  Returns (counts, obj); outputs are host numpy arrays unless
        device tensors are passed in `counts` / `obj`."""
        cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        n = len(cfgs)
        ttl_arr = None if ttl is None else np.ascontiguousarray(ttl, np.uint32)
        if ttl_arr is not None and (ttl_arr.ndim != 2 or ttl_arr.shape[1] != trace.K + 1):
            raise ValueError(f"ttl table must be [n_tuner][K+1] = [*][{trace.K + 1}]")
        n_tuner = 0 if ttl_arr is None else int(ttl_arr.shape[0])
        on_dev = False
        if counts is None and obj is None:
            counts = np.zeros(n, COUNTS_DTYPE)
            obj = np.zeros((n, 3), np.float64)
        pc, po, on_dev = _check_outputs(counts, obj, n)
        m = model.c()
        self._check(self._L.kareto_eval_grid(self._h, trace._h, cfgs.ctypes.data if n else None, n,
                                             None if ttl_arr is None else ttl_arr.ctypes.data, n_tuner,
                                             ctypes.byref(m), pc, po, int(on_dev)), "eval_grid")
        return counts, obj

    def grid(self, cfgs: np.ndarray, ttl=None, n_groups: int | None = None) -> "Grid":
        """kareto_grid_create: a configuration grid prepared once for repeated evaluation."""
        cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        ttl_arr = None if ttl is None else np.ascontiguousarray(ttl, np.uint32)
        if ttl_arr is not None:
            if ttl_arr.ndim != 2:
                raise ValueError("ttl table must be [n_tuner][K+1]")
            n_groups = int(ttl_arr.shape[1])
        if n_groups is None:
            raise ValueError("n_groups (K+1) is needed when no TTL table is given")
        h = ctypes.c_void_p()
        self._check(self._L.kareto_grid_create(self._h, cfgs.ctypes.data if len(cfgs) else None, len(cfgs),
                                               None if ttl_arr is None else ttl_arr.ctypes.data,
                                               0 if ttl_arr is None else int(ttl_arr.shape[0]), int(n_groups),
                                               ctypes.byref(h)), "grid_create")
        return Grid(self, h, len(cfgs))

    def eval_prepared(self, trace: "Trace", grid: "Grid", model: Model, counts=None, obj=None):
        """kareto_eval_grid_prepared: kareto_eval_grid over a prepared grid."""
        n = grid.n
        if counts is None and obj is None:
            counts = np.zeros(n, COUNTS_DTYPE)
            obj = np.zeros((n, 3), np.float64)
        pc, po, on_dev = _check_outputs(counts, obj, n)
        m = model.c()
        self._check(self._L.kareto_eval_grid_prepared(self._h, trace._h, grid._h, ctypes.byref(m), pc, po,
                                                      int(on_dev)), "eval_grid_prepared")
        return counts, obj

    def pareto_prepared(self, obj, grid: "Grid", tau_e: float | None = 0.05, status=None):
        """kareto_pareto_prepared -> (status uint8 [n], n_frontier)."""
        n = grid.n
        po, dev = _ptr(obj)
        if status is None:
            status = np.zeros(n, np.uint8)
        ps, sdev = _ptr(status)
        assert sdev == dev, "obj and status must both be host or both be device buffers"
        pr = PruneC(1 if tau_e is not None else 0, float(tau_e) if tau_e is not None else 0.0)
        nf = ctypes.c_int64()
        self._check(self._L.kareto_pareto_prepared(self._h, po, grid._h, ctypes.byref(pr), ps, ctypes.byref(nf),
                                                   int(dev)), "pareto_prepared")
        return status, int(nf.value)

    def pareto(self, obj, cfgs: np.ndarray | None = None, tau_e: float | None = 0.05, status=None):
        """kareto_pareto -> (status uint8 [n]: 2 pruned / 1 frontier / 0 dominated, n_frontier)."""
        n = int(obj.shape[0])
        po, dev = _ptr(obj)
        if status is None:
            status = np.zeros(n, np.uint8)
        ps, sdev = _ptr(status)
        assert sdev == dev, "obj and status must both be host or both be device buffers"
        pr = PruneC(1 if tau_e is not None else 0, float(tau_e) if tau_e is not None else 0.0)
        cf = None if cfgs is None else np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        nf = ctypes.c_int64()
        self._check(self._L.kareto_pareto(self._h, po, None if cf is None else cf.ctypes.data, n, ctypes.byref(pr),
                                          ps, ctypes.byref(nf), int(dev)), "pareto")
        return status, int(nf.value)

    def hypervolume(self, obj, ref, mask=None) -> float:
        """kareto_hypervolume: exact 3-D hypervolume of the (masked) points w.r.t. ref (row f1)."""
        n = int(obj.shape[0])
        po, dev = _ptr(obj)
        pm, mdev = _ptr(mask)
        assert mask is None or mdev == dev, "obj and mask must both be host or both be device buffers"
        r = (ctypes.c_double * 3)(*[float(v) for v in ref])
        hv = ctypes.c_double()
        self._check(self._L.kareto_hypervolume(self._h, po, pm, n, ctypes.byref(r), ctypes.byref(hv), int(dev)),
                    "hypervolume")
        return float(hv.value)

    def search(self, trace: "Trace", model: Model, d_range, t_range, hbm_gb: float, tau_e=0.05, tau_perf=0.05,
               tau_cost=0.02, policy=LRU, max_rounds=0, cap=1 << 16, expand_ttl=False):
        """kareto_search: Alg. 1 adaptive Pareto exploration (row f1).  d_range / t_range =
        (min, max, step) in GB / s.  Returns (points [SEARCH_POINT_DTYPE], truncated)."""
        p = SearchParamsC(float(hbm_gb), *[int(v) for v in d_range], *[int(v) for v in t_range], float(tau_e),
                          float(tau_perf), float(tau_cost), int(policy), int(max_rounds), int(bool(expand_ttl)), 0)
        out = np.zeros(int(cap), SEARCH_POINT_DTYPE)
        n, tr_ = ctypes.c_int64(), ctypes.c_int32()
        m = model.c()
        self._check(self._L.kareto_search(self._h, trace._h, ctypes.byref(p), ctypes.byref(m),
                                          out.ctypes.data if cap else None, int(cap), ctypes.byref(n),
                                          ctypes.byref(tr_)), "search")
        return out[:n.value].copy(), bool(tr_.value)


    # ---- row f2: Alg. 2 group TTLs
    def ttl_roi(self, trace: "Trace"):
        """kareto_ttl_roi -> (t_roi, H at t_roi, C at t_roi), each [K+1]."""
        G = trace.K + 1
        t, h, c = np.zeros(G, np.uint32), np.zeros(G, np.uint64), np.zeros(G, np.uint64)
        self._check(self._L.kareto_ttl_roi(self._h, trace._h, t.ctypes.data, h.ctypes.data, c.ctypes.data), "ttl_roi")
        return t, h, c

    def ttl_eval(self, trace: "Trace", ttl):
        """kareto_ttl_eval: (sum H, sum C) of each TTL vector in ttl [n][K+1] (ms)."""
        ttl = np.ascontiguousarray(np.atleast_2d(ttl), np.uint32)
        n = ttl.shape[0]
        h, c = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        self._check(self._L.kareto_ttl_eval(self._h, trace._h, ttl.ctypes.data if n else None, n,
                                            h.ctypes.data if n else None, c.ctypes.data if n else None), "ttl_eval")
        return h, c

    def ttl_allocate(self, trace: "Trace", budget: int, seed: int = 0):
        """kareto_ttl_allocate -> dict(t, hits, cost, t_roi, t_init)."""
        G = trace.K + 1
        t, tr_, ti = np.zeros(G, np.uint32), np.zeros(G, np.uint32), np.zeros(G, np.uint32)
        h, c = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self._L.kareto_ttl_allocate(self._h, trace._h, int(budget), int(seed), t.ctypes.data,
                                                ctypes.byref(h), ctypes.byref(c), tr_.ctypes.data, ti.ctypes.data),
                    "ttl_allocate")
        return dict(t=t, hits=int(h.value), cost=int(c.value), t_roi=tr_, t_init=ti)


    # ---- row f4: trace analytics (X5, X6)
    def analytics(self, trace: "Trace", n_pts: int = 101, series: bool = True) -> dict:
        """kareto_trace_analytics -> dict of the scalars, 'lorenz' [n_pts] and (series=True)
        'cumulative' / 'active' [R]."""
        a = AnalyticsC()
        lor = np.zeros(n_pts, np.float64)
        cum = np.zeros(trace.R, np.int64) if series else None
        act = np.zeros(trace.R, np.int64) if series else None
        self._check(self._L.kareto_trace_analytics(self._h, trace._h, ctypes.byref(a),
                                                   lor.ctypes.data if n_pts else None, int(n_pts),
                                                   None if cum is None else cum.ctypes.data,
                                                   None if act is None else act.ctypes.data), "trace_analytics")
        d = {f: getattr(a, f) for f, _ in AnalyticsC._fields_}
        d.update(lorenz=lor, cumulative=cum, active=act)
        return d


    # ---- row f3: queue-coupled disk prefetch, TTFT distribution
    def eval_queue(self, trace: "Trace", cfgs: np.ndarray, model: Model, ttl=None) -> np.ndarray:
        """kareto_eval_queue -> QUEUE_DTYPE [n]."""
        cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
        n = len(cfgs)
        ttl_arr, n_tuner = None, 0
        if ttl is not None:
            ttl_arr = np.ascontiguousarray(ttl, np.uint32)
            n_tuner = ttl_arr.shape[0]
        out = np.zeros(n, QUEUE_DTYPE)
        m = model.c()
        self._check(self._L.kareto_eval_queue(self._h, trace._h, cfgs.ctypes.data if n else None, n,
                                              None if ttl_arr is None else ttl_arr.ctypes.data, n_tuner,
                                              ctypes.byref(m), out.ctypes.data if n else None), "eval_queue")
        return out


class Grid:
    """kareto_grid handle (free before its context is closed)."""

    def __init__(self, ctx: "Context", h, n: int):
        self.ctx, self._h, self.n = ctx, h, n

    def free(self):
        if getattr(self, "_h", None) and getattr(self.ctx, "_h", None):
            self.ctx._L.kareto_grid_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Trace:
    """kareto_trace handle (device-resident)."""

    def __init__(self, ctx: Context, h):
        self.ctx, self._h = ctx, h
        info = TraceInfo()
        st = ctx._L.kareto_trace_stats(h, ctypes.byref(info), None, None)
        ctx._check(st, "trace_stats")
        self.R, self.N, self.U = info.n_requests, info.n_accesses, info.n_unique
        self.span_ms, self.Ltok, self.O = info.span_ms, info.input_tokens, info.output_tokens
        self.K, self.max_blocks = info.top_k, info.max_blocks_per_request
        self.U_g = np.zeros(self.K + 1, np.int64)
        self.reuse_g = np.zeros(self.K + 1, np.int64)
        ctx._L.kareto_trace_stats(h, ctypes.byref(info), self.U_g.ctypes.data, self.reuse_g.ctypes.data)
        v = [ctypes.c_int64() for _ in range(4)]
        ctx._check(ctx._L.kareto_trace_shard(h, *[ctypes.byref(x) for x in v]), "trace_shard")
        # requests [req_lo, req_hi) and positions [pos_lo, pos_hi) held (whole trace: [0, R), [0, N))
        self.req_lo, self.req_hi, self.pos_lo, self.pos_hi = (int(x.value) for x in v)

    def export(self, which: int) -> np.ndarray:
        n = self.pos_hi - self.pos_lo
        if which == X_HASH:
            out = np.zeros(n, np.uint64)
        elif which in (X_PREV, X_DELTA, X_REQ, X_DEPTH):
            out = np.zeros(n, np.uint32)
        elif which == X_GROUP:
            out = np.zeros(self.R, np.uint16)
        elif which == X_START:
            out = np.zeros(self.R + 1, np.uint32)
        else:
            raise ValueError(which)
        if out.size:
            self.ctx._check(self.ctx._L.kareto_trace_export(self.ctx._h, self._h, which, out.ctypes.data), "export")
        return out

    def free(self):
        if getattr(self, "_h", None):
            self.ctx._L.kareto_trace_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Host-only: the shard [lo, hi) of n configurations evaluated by `rank` (no GPU needed)."""
    L = load_library()
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    st = L.kareto_shard_range(n, rank, world, ctypes.byref(lo), ctypes.byref(hi))
    if st != OK:
        raise KaretoError(st, "shard_range")
    return int(lo.value), int(hi.value)


def shard_bounds(cfgs: np.ndarray, world: int, ttl=None, n_groups: int = 1) -> np.ndarray:
    """Host-only: the cost-balanced shard bounds [world + 1] kareto_eval_grid uses (no GPU)."""
    L = load_library()
    cfgs = np.ascontiguousarray(cfgs, CONFIG_DTYPE)
    ttl_arr = None if ttl is None else np.ascontiguousarray(ttl, np.uint32)
    if ttl_arr is not None:
        n_groups = int(ttl_arr.shape[1])
    out = np.zeros(world + 1, np.int64)
    st = L.kareto_shard_bounds(cfgs.ctypes.data if len(cfgs) else None, len(cfgs),
                               None if ttl_arr is None else ttl_arr.ctypes.data,
                               0 if ttl_arr is None else int(ttl_arr.shape[0]), n_groups, world, out.ctypes.data)
    if st != OK:
        raise KaretoError(st, "shard_bounds")
    return out


def time_slices(s, world: int) -> np.ndarray:
    """Host-only: request bounds [world + 1] of the time-sharded load (kareto_time_slices)."""
    L = load_library()
    s = np.ascontiguousarray(s, np.uint32)
    out = np.zeros(world + 1, np.int64)
    st = L.kareto_time_slices(s.ctypes.data, len(s) - 1, world, out.ctypes.data)
    if st != OK:
        raise KaretoError(st, "time_slices")
    return out


def hash_owner(block_hash: int, world: int) -> int:
    """Host-only: the rank owning a block hash in the time-sharded exchange (kareto_hash_owner)."""
    return int(load_library().kareto_hash_owner(int(block_hash), world))


def load_trace(ctx: Context, *a, **k) -> Trace:
    return ctx.load_trace(*a, **k)


def eval_grid(ctx: Context, trace: Trace, cfgs, model: Model, ttl=None, **k):
    return ctx.eval_grid(trace, cfgs, model, ttl, **k)


def pareto(ctx: Context, obj, cfgs=None, tau_e=0.05, **k):
    return ctx.pareto(obj, cfgs, tau_e, **k)

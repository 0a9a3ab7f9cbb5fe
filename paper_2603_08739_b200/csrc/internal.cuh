// internal.cuh -- shared internals of libkareto (context, device arena, errors, pass timing).
// Not part of the ABI; see include/kareto.h.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <string>
#include <vector>

#include "kareto.h"

namespace kareto {

constexpr uint32_t kNone = 0xFFFFFFFFu;  // "no previous access" / "first access" / infinity
// internal status (never returned by the ABI): kareto_load_trace re-runs the load with K2's full sort
constexpr kareto_status KARETO_RETRY_FULL_SORT = (kareto_status)100;
constexpr int kMaxPasses = 64;

struct PassAcc {
  char name[24];
  double ms;
  int launches;
  int own;
};

// dlopen'ed NCCL entry points (loaded by ctx.cu)
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  // used by the time-sharded load (optional: absent => KARETO_E_NCCL there)
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

}  // namespace kareto

struct kareto_loopback;  // in-process rank group (comm.cu)

struct kareto_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  void *nccl_comm = nullptr;  // ncclComm_t
  kareto::NcclApi *nccl = nullptr;
  kareto_loopback *loop = nullptr;  // world > 1 without NCCL: ranks are threads of this process
  cudaMemPool_t pool = nullptr;
  int num_sms = 148;
  size_t l2_bytes = 0;
  std::string err;
  // profiling
  bool profiling = false;
  std::vector<kareto::PassAcc> passes;
  struct Pending {
    int idx;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  int64_t own_launches = 0;
  // K2 bucket-link pairs and records kept between loads (20 B per access, grown on demand,
  // freed by kareto_destroy)
  void *k2_scratch = nullptr;
  size_t k2_scratch_bytes = 0;
  // staging buffer for host-resident tokens / block hashes (kept between loads: a fresh multi-GB
  // pool allocation per load could not reuse the fragmented free blocks and mapped new memory,
  // ~57 ms per config-4 load with host inputs)
  void *h2d_scratch = nullptr;
  size_t h2d_scratch_bytes = 0;
  bool k2_full = false;  // this load uses the full 32-bit K2 sort (after a bucket-table overflow)
};

struct kareto_trace {
  kareto_ctx *ctx = nullptr;
  cudaStream_t stream = nullptr;  // copy of ctx->stream (trace_free must not touch ctx)
  int64_t R = 0, N = 0, U = 0, span_ms = 1;
  int32_t K = 0, max_blocks = 0;
  int64_t n_runs = 0;          // runs of consecutive previous positions (K3)
  // Time-sharded traces (kareto_load_trace_sharded) hold only the accesses of positions
  // [pos_lo, pos_hi) = the blocks of sorted requests [req_lo, req_hi); per-access arrays are
  // indexed by position - pos_lo.  Whole traces: [0, N), [0, R).
  bool sharded = false;
  int64_t pos_lo = 0, pos_hi = 0, req_lo = 0, req_hi = 0;
  uint64_t Ltok = 0, O = 0;
  // sum_r L_r and sum_r L_r (L_r - 1) / 2 as exact 128-bit values (for P0 = alpha*SL + beta*SQ)
  unsigned __int128 SL = 0, SQ = 0;
  // per request (sorted order) [R] / [R+1]
  int64_t *arr = nullptr;      // arrival ms
  uint32_t *s = nullptr;       // first touch position [R+1]
  uint16_t *grp = nullptr;     // group of request
  uint32_t *inlen = nullptr;   // input tokens L_r (saturated at 2^32-1; flagged)
  uint32_t *outlen = nullptr;  // output tokens o_r
  // per access (touch order) [N]
  uint64_t *hash = nullptr;
  uint32_t *req = nullptr;
  uint32_t *prev = nullptr;
  uint32_t *delta = nullptr;
  uint32_t *depth = nullptr;   // LRU depth d at request start (kNone: first access)
  // K3 runs of a whole trace [n_runs] (j0, L, d0, r): accesses j0 .. j0+L-1 of request r with
  // consecutive previous positions; d_{j0+t} = d0 - t (K4 histograms a run at once, eval.cu)
  uint4 *runs = nullptr;
  bool depth_ready = true;     // false: depth is materialised from runs on first use
  // K6 replay inputs, built on first use (replay.cu)
  uint32_t *blk = nullptr;     // [N] dense block id
  uint16_t *gblk = nullptr;    // [U] group of each block
  uint32_t *arr_rel = nullptr; // [R] arrival - first arrival (ms)
  // group tables (host) [K+1]
  std::vector<int64_t> U_g, reuse_g;
};

namespace kareto {
struct GridPrep;  // eval.cu
}
// A configuration grid prepared for repeated evaluation (kareto_grid_create): eval_grid's
// validation, shard, stack / replay split and device copies (GridPrep), and K8's device copy of
// every configuration with its line-key bit widths.
struct kareto_grid {
  kareto_ctx *ctx = nullptr;
  kareto::GridPrep *prep = nullptr;
  kareto::GridPrep *prep_whole = nullptr;  // built on first use with a time-sharded trace
  int64_t n = 0;
  kareto_config *dall = nullptr;  // [n] device (pool), freed by kareto_grid_free
  int lw[6] = {0, 0, 0, 0, 0, 0};
  bool lw_ok = false;             // the axis / line-key ranges pruning needs
  std::string lw_err;
  // K8a line order per axis (pareto.cu), built on the first pruned selection: the sorted line
  // keys and the configuration permutation depend on the grid alone
  uint64_t *lkey[3] = {nullptr, nullptr, nullptr};
  uint32_t *lidx[3] = {nullptr, nullptr, nullptr};
};

namespace kareto {

// ----------------------------------------------------------------- errors ----
inline kareto_status fail(kareto_ctx *ctx, kareto_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return st;
}

#define KCUDA(ctx, call)                                                                              \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess) {                                                                          \
      kareto_status st_ = (e_ == cudaErrorMemoryAllocation) ? KARETO_E_OOM : KARETO_E_CUDA;           \
      (void)cudaGetLastError();                                                                       \
      return ::kareto::fail(ctx, st_, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    }                                                                                                 \
  } while (0)

#define KTRY(expr)                      \
  do {                                  \
    kareto_status st_ = (expr);         \
    if (st_ != KARETO_OK) return st_;   \
  } while (0)

// allocation from the context's pool (ptr, bytes) on stream st
#define KMALLOC(ctx, ptr, bytes, st) KCUDA(ctx, cudaMallocFromPoolAsync((void **)&(ptr), (bytes), (ctx)->pool, (st)))

// Device bytes a wave of K6 / queue state may take: `frac` of what is free (device + unused pool
// reserve), divided among the loopback ranks sharing this GPU; KARETO_K6_BUDGET (bytes) overrides
// (tests use it to force many waves).  Synchronises the context stream.
kareto_status wave_budget(kareto_ctx *ctx, double frac, double *bytes);
// return the pool's unused reserve to the device (after large transient allocations)
void pool_trim(kareto_ctx *ctx);
// materialise tr->depth from the kept K3 runs if a whole-trace load deferred it (stack_depth.cu)
kareto_status ensure_depth(kareto_ctx *ctx, kareto_trace *tr);

// KARETO_HOSTTIME=1: wall-clock marks (after a stream sync) through a call, to stderr -- shows
// where a step's time goes between the profiled passes (host work, syncs, allocations)
struct HostMarks {
  bool on = getenv("KARETO_HOSTTIME") != nullptr;
  bool nosync = on && getenv("KARETO_HOSTTIME")[0] == '2';  // host timestamps only
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), tl = t0;
  const char *what;
  explicit HostMarks(const char *w) : what(w) {}
  void mark(cudaStream_t st, const char *name) {
    if (!on) return;
    if (!nosync) cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[%s] %-22s +%.3f ms (at %.3f ms)\n", what, name,
            std::chrono::duration<double, std::milli>(t - tl).count(),
            std::chrono::duration<double, std::milli>(t - t0).count());
    tl = t;
  }
};

// ----------------------------------------------------- stream-ordered buffers ----
// Device buffers come from the device's stream-ordered memory pool (cudaMallocFromPoolAsync on
// the context stream, release threshold = unlimited), so repeated loads/evals reuse HBM without
// cudaMalloc/cudaFree synchronisation; the pool is trimmed after the large transient K6 / queue
// allocations (pool_trim), so its unused reserve goes back to the device.
template <typename T>
struct DBuf {
  kareto_ctx *ctx = nullptr;
  T *p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : ctx(o.ctx), p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    release();
    ctx = o.ctx; p = o.p; n = o.n; o.p = nullptr; o.n = 0;
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, ctx->stream);
    p = nullptr;
    n = 0;
  }
  T *detach() { T *q = p; p = nullptr; n = 0; return q; }
  kareto_status alloc(kareto_ctx *c, size_t count) {
    release();
    ctx = c;
    n = count;
    size_t bytes = (count ? count : 1) * sizeof(T);
    cudaError_t e = cudaMallocFromPoolAsync((void **)&p, bytes, c->pool, c->stream);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      p = nullptr;
      return fail(c, KARETO_E_OOM, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    }
    return KARETO_OK;
  }
  kareto_status zero() {
    cudaError_t e = cudaMemsetAsync(p, 0, (n ? n : 1) * sizeof(T), ctx->stream);
    if (e != cudaSuccess) return fail(ctx, KARETO_E_CUDA, "memset: %s", cudaGetErrorString(e));
    return KARETO_OK;
  }
};

// -------------------------------------------------------------- pass timing ----
// Scope object bracketing one pass (one or more launches) with CUDA events on the
// context stream when profiling is on.  Own-kernel launches are always counted.
struct Pass {
  kareto_ctx *ctx;
  int idx = -1;
  cudaEvent_t a = nullptr, b = nullptr;
  Pass(kareto_ctx *c, const char *name, int own, int launches);
  ~Pass();
};

// Resolve pending pass events into the accumulators (after the call's final sync).
void flush_pass_times(kareto_ctx *ctx);

// final synchronisation of a call: stream sync + launch error check
kareto_status sync(kareto_ctx *ctx, const char *what);

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 1 << 30) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

// ----------------------------------------------------------- device helpers ----
// splitmix64 finaliser (R2); this library's own copy.
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kChainR = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kSaltC = 0x243F6A8885A308D3ULL;

// ------------------------------------------------------------ collectives (comm.cu) ----
// Every rank of ctx calls these collectively, in the same order.  Buffers are device
// buffers of the context device unless named *_host.  World == 1: plain local copies.
kareto_status coll_allgather(kareto_ctx *ctx, const void *send, void *recv, size_t bytes);
kareto_status coll_allgather_host(kareto_ctx *ctx, const void *send, void *recv, size_t bytes);
kareto_status coll_allreduce_u64(kareto_ctx *ctx, unsigned long long *buf, size_t n);  // in place, sum
// send_off / recv_off: [world + 1] byte offsets; rank r's segment [off[r], off[r+1]) goes to /
// comes from rank r.  Receive sizes must match what the peers send.
kareto_status coll_alltoallv(kareto_ctx *ctx, const void *send, const std::vector<size_t> &send_off, void *recv,
                             const std::vector<size_t> &recv_off);


}  // namespace kareto

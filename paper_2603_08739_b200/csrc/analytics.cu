// analytics.cu -- trace analytics of row f4 from the resident trace (DESIGN R47-R48):
//   X6 reuse skew: hits per block, the Lorenz curve of hits over blocks sorted by
//      hits, and the fewest top blocks holding >= 90% of the hits;
//   X5 oracle-TTL footprint: after each request, the distinct blocks seen so far and
//      the blocks whose next access is in a later request.
// B200 design: hits per dense block id (one atomic per reuse access; ids from the K6 prepare
// pass), a CUB descending sort + scan for the Lorenz curve; the footprint is two difference
// arrays over requests (+1 at a block's first request; +1 / -1 over [request of the previous
// access, request of this access) for every reuse) and two CUB scans.
#include <cub/cub.cuh>

#include <vector>

#include "internal.cuh"
#include "replay.cuh"

namespace kareto {

__global__ void k_block_hits(uint64_t N, const uint32_t *__restrict__ blk, const uint32_t *__restrict__ prev,
                             uint32_t *__restrict__ cnt) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x)
    if (prev[j] != kNone) atomicAdd(&cnt[blk[j]], 1u);
}

__global__ void k_widen(const uint32_t *__restrict__ a, uint64_t n, unsigned long long *__restrict__ b) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// smallest k >= 1 with 10 * pre[k-1] >= 9 * T (pre inclusive over the descending hits)
__global__ void k_k90(const unsigned long long *__restrict__ pre, uint64_t U, unsigned long long *__restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  const unsigned __int128 T = pre[U - 1];
  uint64_t lo = 1, hi = U;
  while (lo < hi) {
    const uint64_t m = (lo + hi) / 2;
    if ((unsigned __int128)10 * pre[m - 1] >= 9 * T) hi = m; else lo = m + 1;
  }
  out[0] = lo;
}

__global__ void k_lorenz(const unsigned long long *__restrict__ pre, uint64_t U, int n, double *__restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double T = (double)pre[U - 1];
  const uint64_t k = (uint64_t)(((unsigned __int128)i * U + (uint64_t)(n - 2)) / (uint64_t)(n - 1));  // ceil
  y[i] = (k == 0 || T == 0) ? 0.0 : (double)pre[k - 1] / T;
}

__global__ void k_fp_diff(uint64_t N, const uint32_t *__restrict__ prev, const uint32_t *__restrict__ req,
                          unsigned long long *__restrict__ cumd, unsigned long long *__restrict__ actd) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = prev[j], r = req[j];
    if (p == kNone) {
      atomicAdd(&cumd[r], 1ull);
    } else {
      atomicAdd(&actd[req[p]], 1ull);
      atomicAdd(&actd[r], ~0ull);  // -1 (two's complement)
    }
  }
}

__global__ void k_first_max(const long long *__restrict__ a, int64_t n, const long long *__restrict__ mx,
                            unsigned long long *__restrict__ first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (a[i] == *mx) atomicMin(first, (unsigned long long)i);
}

template <typename F>
static kareto_status cub_go(kareto_ctx *ctx, DBuf<uint8_t> &tmp, F &&f) {
  size_t bytes = 0;
  KCUDA(ctx, f((void *)nullptr, bytes));
  if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
  size_t b2 = tmp.n;
  KCUDA(ctx, f((void *)tmp.p, b2));
  return KARETO_OK;
}

static kareto_status analytics(kareto_ctx *ctx, kareto_trace *tr, kareto_analytics *out, double *lorenz, int n_pts,
                               int64_t *cumulative, int64_t *active) {
  if (!out || n_pts < 0 || n_pts == 1 || (n_pts > 0 && !lorenz))
    return fail(ctx, KARETO_E_INVALID, "trace_analytics: bad arguments (n_pts must be 0 or >= 2)");
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const uint64_t N = (uint64_t)tr->N, U = (uint64_t)tr->U;
  const int64_t R = tr->R;
  memset(out, 0, sizeof(*out));
  out->unique_blocks = (int64_t)U;
  out->frac_90 = 1.0;
  DBuf<uint8_t> tmp;
  // ---- X6
  if (N > 0 && U > 0) {
    KTRY(replay_prepare(ctx, tr));  // dense block ids
    Pass ps(ctx, "F4_skew", 1, 4);
    DBuf<uint32_t> cnt, cs;
    DBuf<unsigned long long> w, pre, k90;
    KTRY(cnt.alloc(ctx, U)); KTRY(cs.alloc(ctx, U)); KTRY(w.alloc(ctx, U)); KTRY(pre.alloc(ctx, U));
    KTRY(k90.alloc(ctx, 1));
    KTRY(cnt.zero());
    k_block_hits<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->blk, tr->prev, cnt.p);
    KTRY(cub_go(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortKeysDescending(t, b, cnt.p, cs.p, (int64_t)U, 0, 32, st);
    }));
    k_widen<<<grid_for(U, 256, 8 * sms), 256, 0, st>>>(cs.p, U, w.p);
    KTRY(cub_go(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceScan::InclusiveSum(t, b, w.p, pre.p, (int64_t)U, st); }));
    unsigned long long T = 0;
    KCUDA(ctx, cudaMemcpyAsync(&T, pre.p + (U - 1), 8, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    out->total_hits = (int64_t)T;
    if (T > 0) {
      k_k90<<<1, 1, 0, st>>>(pre.p, U, k90.p);
      unsigned long long k = 0;
      KCUDA(ctx, cudaMemcpyAsync(&k, k90.p, 8, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      out->blocks_90 = (int64_t)k;
      out->frac_90 = (double)k / (double)U;
    } else {
      out->blocks_90 = (int64_t)U;
    }
    if (n_pts > 0) {
      DBuf<double> y;
      KTRY(y.alloc(ctx, n_pts));
      k_lorenz<<<grid_for(n_pts, 256), 256, 0, st>>>(pre.p, U, n_pts, y.p);
      KCUDA(ctx, cudaMemcpyAsync(lorenz, y.p, 8 * (size_t)n_pts, cudaMemcpyDeviceToHost, st));
    }
  } else if (n_pts > 0) {
    for (int i = 0; i < n_pts; i++) lorenz[i] = 0.0;
  }
  // ---- X5
  if (R > 0) {
    Pass ps(ctx, "F4_footprint", 1, 2);
    DBuf<unsigned long long> cumd, actd, cum, act, first;
    DBuf<long long> mx;
    KTRY(cumd.alloc(ctx, R)); KTRY(actd.alloc(ctx, R)); KTRY(cum.alloc(ctx, R)); KTRY(act.alloc(ctx, R));
    KTRY(first.alloc(ctx, 1)); KTRY(mx.alloc(ctx, 1));
    KTRY(cumd.zero()); KTRY(actd.zero());
    KCUDA(ctx, cudaMemsetAsync(first.p, 0xFF, 8, st));
    if (N > 0) k_fp_diff<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->prev, tr->req, cumd.p, actd.p);
    KTRY(cub_go(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceScan::InclusiveSum(t, b, cumd.p, cum.p, R, st); }));
    KTRY(cub_go(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceScan::InclusiveSum(t, b, actd.p, act.p, R, st); }));
    const long long *actl = reinterpret_cast<const long long *>(act.p);
    KTRY(cub_go(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceReduce::Max(t, b, actl, mx.p, R, st); }));
    k_first_max<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(actl, R, mx.p, first.p);
    long long hm = 0;
    unsigned long long hf = 0;
    KCUDA(ctx, cudaMemcpyAsync(&hm, mx.p, 8, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaMemcpyAsync(&hf, first.p, 8, cudaMemcpyDeviceToHost, st));
    if (cumulative) KCUDA(ctx, cudaMemcpyAsync(cumulative, cum.p, 8 * R, cudaMemcpyDeviceToHost, st));
    if (active) KCUDA(ctx, cudaMemcpyAsync(active, act.p, 8 * R, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    out->peak_active = hm;
    out->peak_active_request = (int64_t)hf;
    unsigned long long last = 0;
    KCUDA(ctx, cudaMemcpyAsync(&last, cum.p + (R - 1), 8, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    out->final_cumulative = (int64_t)last;
  }
  return sync(ctx, "trace analytics");
}

}  // namespace kareto

extern "C" kareto_status kareto_trace_analytics(kareto_ctx *ctx, const kareto_trace *tr, kareto_analytics *out,
                                                double *lorenz, int32_t n_pts, int64_t *cumulative, int64_t *active) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  if (tr && tr->sharded)
    return kareto::fail(ctx, KARETO_E_UNSUPPORTED, "%s needs the whole trace (not a time shard)", "kareto_trace_analytics");
  cudaSetDevice(ctx->device);
  if (!tr) return kareto::fail(ctx, KARETO_E_INVALID, "trace_analytics: null trace");
  kareto_status s = kareto::analytics(ctx, const_cast<kareto_trace *>(tr), out, lorenz, n_pts, cumulative, active);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

// stack_depth.cu -- row a4, K3: exact LRU stack depth of every reuse access.
//
// The pre-request LRU depth of access j of request r with previous access p is
//     d_j = s_r - p - A(p, s_r),   A(y, s) = #{ i < s : prev[i] >= y }
// (live positions in [p, s_r); the O2 oracle computes the same with
// a sequential Fenwick tree).  A is an offline 2-D dominance count.
//
// Run compression (exact for any trace): inside one request, a maximal run
// of consecutive positions j0..j0+L-1 whose previous positions are consecutive,
// prev[j0+t] = p0 + t, has
//   (i)  one A for the whole run: A(y) - A(y+1) = [y re-touched before s_r], and no prev
//        value y of the run is re-touched before s_r (it is the LAST earlier occurrence);
//   (ii) one kill interval [p0, p0+L) (the y values it re-touches) at one time (its request).
// Kill intervals are disjoint (each position is re-touched at most once) and an interval
// that contains a query's p0 is killed at or after the query's request.  Hence
//     A(run q) = sum of L' over runs q' of EARLIER requests with p0' > p0(q),
// a weighted 2-D dominance count over runs -- ~2-3 runs per request instead of ~80
// accesses.  It is solved by an MSD radix partition with counting (items: per request, its
// query items then its weighted point items; each level adds the weight of earlier points
// of the segment with a larger digit) and a per-segment Fenwick finish; d is then expanded
// back to every access of the run.
//
// Item = uint2 {y, w}: query: w = running count (< 2^31); point: w = 0x80000000 | L.
#include <cub/cub.cuh>

#include "trace_load.cuh"

namespace kareto {

constexpr int SD_WARPS = 8;
constexpr int SD_CHUNKS = 16;                          // chunks of 32 items per warp per tile
constexpr int SD_TILE = SD_WARPS * SD_CHUNKS * 32;     // 4096 items per tile
constexpr int SD_LOCAL_BITS = 11;
constexpr uint32_t kPointBit = 0x80000000u;

__device__ __forceinline__ bool is_point(uint32_t w) { return (w & kPointBit) != 0; }
__device__ __forceinline__ uint32_t pweight(uint32_t w) { return is_point(w) ? (w & ~kPointBit) : 0u; }

struct Tile {
  uint32_t seg, t;   // segment, local tile index
};

struct PassArgs {
  const uint2 *in;
  const Tile *tiles;
  const uint64_t *seg_start;   // [nseg] start offsets of segments in `in`
  const uint64_t *seg_len;     // [nseg]
  const uint32_t *seg_tile0;   // [nseg] first global tile of the segment
  const uint32_t *seg_ntiles;  // [nseg]
  int shift, bits;             // digit = (y >> shift) & (2^bits - 1)
  uint32_t *hist_all, *hist_pts;     // [tiles * bins] layout tile0*bins + d*ntiles + t
  unsigned long long *seg_tot;       // [nseg * bins]
  const uint32_t *off_all, *off_pts; // exclusive sums of the two histograms
  uint2 *out;
};

__device__ __forceinline__ void tile_geometry(const PassArgs &a, uint32_t bid, uint32_t &seg, uint32_t &t,
                                              uint64_t &beg, uint64_t &end, uint32_t &tile0, uint32_t &ntiles) {
  Tile td = a.tiles[bid];
  seg = td.seg; t = td.t;
  if (seg == 0xFFFFFFFFu) { beg = end = 0; tile0 = ntiles = 0; return; }
  tile0 = a.seg_tile0[seg]; ntiles = a.seg_ntiles[seg];
  uint64_t s0 = a.seg_start[seg], L = a.seg_len[seg];
  beg = s0 + (uint64_t)t * SD_TILE;
  uint64_t e = s0 + (uint64_t)(t + 1) * SD_TILE;
  end = e < s0 + L ? e : s0 + L;
}

// ---- run extraction: flags were written by K2 (k_access_info); runs listed by CUB select
// (run_start / req / prev are indexed by local position; req holds global request ids,
// r - req_base indexes s, whose values are global positions: local = s - pos_base)
__global__ void k_run_info(const uint32_t *__restrict__ run_start, const int *__restrict__ m_ptr, uint64_t N,
                           const uint32_t *__restrict__ req, uint32_t req_base, const uint32_t *__restrict__ s,
                           uint32_t pos_base, const uint32_t *__restrict__ prev, uint32_t *__restrict__ run_req,
                           uint32_t *__restrict__ run_len, uint32_t *__restrict__ run_p0) {
  const int M = *m_ptr;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < M; q += gridDim.x * blockDim.x) {
    uint32_t j0 = run_start[q];
    uint32_t r = req[j0] - req_base;
    uint32_t nxt = q + 1 < M ? run_start[q + 1] : (uint32_t)N;
    uint32_t rend = s[r + 1] - pos_base;
    run_req[q] = r;
    run_len[q] = (nxt < rend ? nxt : rend) - j0;
    run_p0[q] = prev[j0];
  }
}

// items of request r occupy [2 q0, 2 q0 + 2 nr): its nr queries, then its nr weighted points
__global__ void k_run_items(const int *__restrict__ m_ptr, const uint32_t *__restrict__ run_req,
                            const uint32_t *__restrict__ run_len, const uint32_t *__restrict__ run_p0,
                            uint2 *__restrict__ items) {
  const int M = *m_ptr;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < M; q += gridDim.x * blockDim.x) {
    uint32_t r = run_req[q];
    // a request has few runs: short linear scans (coalesced neighbours), binary search beyond
    int q0 = q, steps = 0;  // first run of request r
    while (q0 > 0 && run_req[q0 - 1] == r && steps < 8) { q0--; steps++; }
    if (q0 > 0 && run_req[q0 - 1] == r) {
      int lo = 0, hi = q0;
      while (lo < hi) { int m = (lo + hi) >> 1; if (run_req[m] >= r) hi = m; else lo = m + 1; }
      q0 = lo;
    }
    int q1 = q + 1;  // one past the last run of request r
    steps = 0;
    while (q1 < M && run_req[q1] == r && steps < 8) { q1++; steps++; }
    if (q1 < M && run_req[q1] == r) {
      int lo = q1, hi = M;
      while (lo < hi) { int m = (lo + hi) >> 1; if (run_req[m] > r) hi = m; else lo = m + 1; }
      q1 = lo;
    }
    int nr = q1 - q0;
    uint32_t p0 = run_p0[q];
    items[q + q0] = make_uint2(p0, 0u);
    items[q + q0 + nr] = make_uint2(p0, kPointBit | run_len[q]);
  }
}

// ---- upsweep: per-tile digit histograms (item counts, point weights) + segment totals
__global__ void __launch_bounds__(SD_WARPS * 32) k_sd_upsweep(PassArgs a) {
  __shared__ uint32_t h_all[256], h_pts[256];
  const int bins = 1 << a.bits;
  for (int i = threadIdx.x; i < bins; i += blockDim.x) { h_all[i] = 0; h_pts[i] = 0; }
  __syncthreads();
  uint32_t seg, t, tile0, ntiles;
  uint64_t beg, end;
  tile_geometry(a, blockIdx.x, seg, t, beg, end, tile0, ntiles);
  if (seg == 0xFFFFFFFFu) return;  // unused tile slot (upper-bound grid)
  for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    uint2 it = a.in[i];
    uint32_t d = (it.x >> a.shift) & (bins - 1);
    atomicAdd(&h_all[d], 1u);
    if (is_point(it.y)) atomicAdd(&h_pts[d], pweight(it.y));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += blockDim.x) {
    size_t idx = (size_t)tile0 * bins + (size_t)d * ntiles + t;
    a.hist_all[idx] = h_all[d];
    a.hist_pts[idx] = h_pts[d];
    if (h_all[d]) atomicAdd(&a.seg_tot[(size_t)seg * bins + d], (unsigned long long)h_all[d]);
  }
}

// ---- downsweep: stable scatter by digit + weighted query contributions
__global__ void __launch_bounds__(SD_WARPS * 32) k_sd_downsweep(PassArgs a) {
  __shared__ uint32_t run_all[SD_WARPS][256];
  __shared__ uint32_t run_pts[SD_WARPS][256];
  __shared__ uint32_t suf[SD_WARPS][256];
  const int bins = 1 << a.bits;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t seg, t, tile0, ntiles;
  uint64_t beg, end;
  tile_geometry(a, blockIdx.x, seg, t, beg, end, tile0, ntiles);
  if (seg == 0xFFFFFFFFu) return;
  const uint64_t wbeg = beg + (uint64_t)wid * SD_CHUNKS * 32;
  for (int d = lane; d < bins; d += 32) { run_all[wid][d] = 0; run_pts[wid][d] = 0; }
  __syncwarp();
  for (int c = 0; c < SD_CHUNKS; c++) {
    uint64_t i = wbeg + (uint64_t)c * 32 + lane;
    if (i < end) {
      uint2 it = a.in[i];
      uint32_t d = (it.x >> a.shift) & (bins - 1);
      atomicAdd(&run_all[wid][d], 1u);
      if (is_point(it.y)) atomicAdd(&run_pts[wid][d], pweight(it.y));
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += blockDim.x) {
    size_t idx = (size_t)tile0 * bins + (size_t)d * ntiles + t;
    size_t idx0 = (size_t)tile0 * bins + (size_t)d * ntiles;
    uint32_t ra = a.off_all[idx];
    uint32_t rp = a.off_pts[idx] - a.off_pts[idx0];  // point weight of digit d in earlier tiles of the segment
    for (int w = 0; w < SD_WARPS; w++) {
      uint32_t ca = run_all[w][d], cp = run_pts[w][d];
      run_all[w][d] = ra;
      run_pts[w][d] = rp;
      ra += ca;
      rp += cp;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int c = 0; c < SD_CHUNKS; c++) {
    if (wbeg + (uint64_t)c * 32 >= end) break;  // warp-uniform
    // suf[d] = sum_{d' > d} run_pts[d']
    {
      uint32_t v[8], tot = 0;
      int per = bins > 32 ? bins / 32 : 1;
      int base = lane * per;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        v[k] = (k < per && base + k < bins) ? run_pts[wid][base + k] : 0u;
        tot += v[k];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t o = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += o;
      }
      uint32_t acc = incl - tot;
#pragma unroll
      for (int k = 7; k >= 0; k--) {
        if (k < per && base + k < bins) suf[wid][base + k] = acc;
        acc += v[k];
      }
    }
    __syncwarp();
    uint64_t i = wbeg + (uint64_t)c * 32 + lane;
    bool live = i < end;
    uint2 it = live ? a.in[i] : make_uint2(0, 0);
    uint32_t d = live ? (it.x >> a.shift) & (bins - 1) : 0u;
    uint32_t wp = live ? pweight(it.y) : 0u;
    // weight of earlier lanes' points with a larger digit
    uint32_t intra = 0;
#pragma unroll 8
    for (int b = 0; b < 32; b++) {
      uint32_t db = __shfl_sync(0xffffffffu, d, b);
      uint32_t wb = __shfl_sync(0xffffffffu, wp, b);
      if (b < lane && db > d) intra += wb;
    }
    unsigned lm = __ballot_sync(0xffffffffu, live);
    unsigned same = __match_any_sync(0xffffffffu, live ? d : 0xFFFFFFFFu);
    uint32_t gsum = __reduce_add_sync(same, wp);  // point weight of this digit in the chunk
    if (live) {
      uint32_t pos = run_all[wid][d] + __popc(same & lm & lt);
      uint2 o = it;
      if (!is_point(it.y)) o.y = it.y + suf[wid][d] + intra;
      a.out[pos] = o;
    }
    __syncwarp();
    if (live && (__ffs(same & lm) - 1) == lane) {
      run_all[wid][d] += __popc(same & lm);
      run_pts[wid][d] += gsum;
    }
    __syncwarp();
  }
}

// ---- local pass: one warp per segment of 2^LB consecutive y values; weighted Fenwick in smem.
// A[y] = (count so far) + weight of earlier points of the segment with a larger y.
constexpr int LOCAL_WARPS = 4;
template <int LB>
__global__ void __launch_bounds__(LOCAL_WARPS * 32) k_sd_local(const uint2 *__restrict__ in, const uint64_t *__restrict__ seg_start,
                                                  const uint64_t *__restrict__ seg_len, uint32_t nseg,
                                                  uint32_t *__restrict__ A) {
  constexpr int S = 1 << LB;
  __shared__ uint32_t fw[LOCAL_WARPS][S + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t seg = blockIdx.x * LOCAL_WARPS + wid; seg < nseg; seg += gridDim.x * LOCAL_WARPS) {
    const uint64_t s0 = seg_start[seg], L = seg_len[seg];
    if (L == 0) continue;
    for (int k = lane; k <= S; k += 32) fw[wid][k] = 0;
    __syncwarp();
    uint32_t total = 0;  // weight inserted so far
    for (uint64_t c0 = 0; c0 < L; c0 += 32) {
      bool live = c0 + lane < L;
      uint2 it = live ? in[s0 + c0 + lane] : make_uint2(0, 0);
      uint32_t yl = it.x & (S - 1);
      uint32_t wp = live ? pweight(it.y) : 0u;
      uint32_t intra = 0;
#pragma unroll 8
      for (int b = 0; b < 32; b++) {
        uint32_t yb = __shfl_sync(0xffffffffu, yl, b);
        uint32_t wb = __shfl_sync(0xffffffffu, wp, b);
        if (b < lane && yb > yl) intra += wb;
      }
      if (live && !is_point(it.y)) {
        uint32_t le = 0;  // weight with y' <= yl
        for (int k = (int)yl + 1; k > 0; k -= k & -k) le += fw[wid][k];
        A[it.x] = it.y + (total - le) + intra;
      }
      __syncwarp();
      if (wp)
        for (int k = (int)yl + 1; k <= S; k += k & -k) atomicAdd(&fw[wid][k], wp);
      total += __reduce_add_sync(0xffffffffu, wp);
      __syncwarp();
    }
  }
}

// d_j = s_r - prev_j - A(run) for every access of each run; s_r in the coordinates of prev:
// s[r] - pos_base + y_off.  A warp loads the metadata of 32 runs at once (coalesced; the s / A
// gathers of the 32 runs in flight together), then writes the runs one after the other with
// all lanes (consecutive lanes store consecutive positions).
__global__ void __launch_bounds__(256) k_run_expand(const int *__restrict__ m_ptr, const uint32_t *__restrict__ run_start,
                                                    const uint32_t *__restrict__ run_req,
                                                    const uint32_t *__restrict__ run_len,
                                                    const uint32_t *__restrict__ run_p0,
                                                    const uint32_t *__restrict__ s, uint32_t s_shift,
                                                    const uint32_t *__restrict__ A, uint32_t *__restrict__ depth,
                                                    uint4 *__restrict__ runs_out) {
  const int M = *m_ptr;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int q0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; q0 < M; q0 += nw * 32) {
    const int q = q0 + lane;
    uint32_t j0 = 0, L = 0, base = 0;
    if (q < M) {
      const uint32_t p0 = run_p0[q];
      j0 = run_start[q];
      L = run_len[q];
      const uint32_t r = run_req[q];
      base = s[r] - s_shift - p0 - A[p0];
      if (runs_out) runs_out[q] = make_uint4(j0, L, base, r);
    }
    const int nk = M - q0 < 32 ? M - q0 : 32;
    for (int k = 0; k < nk; k++) {
      const uint32_t jk = __shfl_sync(0xFFFFFFFFu, j0, k), Lk = __shfl_sync(0xFFFFFFFFu, L, k);
      const uint32_t bk = __shfl_sync(0xFFFFFFFFu, base, k);
      if (depth)
        for (uint32_t t = lane; t < Lk; t += 32) depth[jk + t] = bk - t;
    }
  }
}

// ---- run heads: ordered compaction of the K2 run flags (two passes over 1 B per access)
constexpr int CF_THREADS = 256, CF_PER = 64, CF_TILE = CF_THREADS * CF_PER;  // 16384 flags per tile
__device__ __forceinline__ uint32_t nz_bytes(uint32_t w) {  // number of nonzero bytes
  return ((w & 0xFFu) != 0) + ((w & 0xFF00u) != 0) + ((w & 0xFF0000u) != 0) + ((w & 0xFF000000u) != 0);
}
__device__ __forceinline__ void load_flags(const uint8_t *__restrict__ f, uint64_t N, uint64_t p, uint32_t w[16]) {
  if (p + 64 <= N) {
    const uint4 *q = reinterpret_cast<const uint4 *>(f + p);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint4 v = __ldg(q + k);
      w[4 * k] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      uint32_t x = 0;
      for (int b = 0; b < 4; b++) {
        const uint64_t i = p + 4 * k + b;
        if (i < N && f[i]) x |= 0xFFu << (8 * b);
      }
      w[k] = x;
    }
  }
}
__global__ void __launch_bounds__(CF_THREADS) k_flag_count(const uint8_t *__restrict__ f, uint64_t N,
                                                           uint32_t *__restrict__ cnt) {
  typedef cub::BlockReduce<uint32_t, CF_THREADS> Red;
  __shared__ typename Red::TempStorage ts;
  const uint64_t p = (uint64_t)blockIdx.x * CF_TILE + (uint64_t)threadIdx.x * CF_PER;
  uint32_t w[16], c = 0;
  if (p < N) {
    load_flags(f, N, p, w);
#pragma unroll
    for (int k = 0; k < 16; k++) c += nz_bytes(w[k]);
  }
  const uint32_t tot = Red(ts).Sum(c);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(CF_THREADS) k_flag_write(const uint8_t *__restrict__ f, uint64_t N,
                                                           const uint32_t *__restrict__ off,
                                                           uint32_t *__restrict__ out) {
  typedef cub::BlockScan<uint32_t, CF_THREADS> Scan;
  __shared__ typename Scan::TempStorage ts;
  const uint64_t p = (uint64_t)blockIdx.x * CF_TILE + (uint64_t)threadIdx.x * CF_PER;
  uint32_t w[16], c = 0;
  if (p < N) {
    load_flags(f, N, p, w);
#pragma unroll
    for (int k = 0; k < 16; k++) c += nz_bytes(w[k]);
  }
  uint32_t ex;
  Scan(ts).ExclusiveSum(c, ex);
  if (!c) return;
  uint32_t o = off[blockIdx.x] + ex;
  for (int k = 0; k < 16; k++)
    for (int b = 0; b < 4; b++)
      if ((w[k] >> (8 * b)) & 0xFFu) out[o++] = (uint32_t)(p + 4 * k + b);
}

__global__ void k_sd_tiles(uint32_t nseg, const uint64_t *__restrict__ seg_len, const uint32_t *__restrict__ tile0,
                           uint32_t *__restrict__ ntiles_out, Tile *__restrict__ tiles, int write) {
  for (uint32_t sgi = blockIdx.x * blockDim.x + threadIdx.x; sgi < nseg; sgi += gridDim.x * blockDim.x) {
    uint32_t nt = (uint32_t)((seg_len[sgi] + SD_TILE - 1) / SD_TILE);
    if (!write) { ntiles_out[sgi] = nt; continue; }
    for (uint32_t t = 0; t < nt; t++) tiles[tile0[sgi] + t] = Tile{sgi, t};
  }
}

__global__ void k_single_segment(const int *__restrict__ m_ptr, uint64_t *__restrict__ start,
                                 uint64_t *__restrict__ len) {
  start[0] = 0;
  len[0] = 2ull * (uint64_t)(*m_ptr);
}

template <typename F>
static kareto_status cub_tmp(kareto_ctx *ctx, DBuf<uint8_t> &tmp, F &&f) {
  size_t bytes = 0;
  KCUDA(ctx, f((void *)nullptr, bytes));
  if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
  size_t b2 = tmp.n;
  KCUDA(ctx, f((void *)tmp.p, b2));
  return KARETO_OK;
}

// Runs of n accesses: ordered compaction of the run-head flags into rl.run_start; rl.m_dev = M
// on the device (no host round trip).
kareto_status run_list_start(kareto_ctx *ctx, uint64_t N, const uint8_t *run_flag, RunList &rl) {
  cudaStream_t st = ctx->stream;
  DBuf<uint8_t> tmp;
  KTRY(rl.m_dev.alloc(ctx, 1));
  KTRY(rl.run_start.alloc(ctx, N > 0 ? N : 1));  // #runs <= reuse accesses
  if (N == 0) return rl.m_dev.zero();
  Pass ps(ctx, "K3_runs", 1, 2);
  const uint64_t ntile = (N + CF_TILE - 1) / CF_TILE;
  DBuf<uint32_t> cnt, off;
  KTRY(cnt.alloc(ctx, ntile + 1)); KTRY(off.alloc(ctx, ntile + 1));
  KCUDA(ctx, cudaMemsetAsync(cnt.p + ntile, 0, 4, st));
  k_flag_count<<<(unsigned)ntile, CF_THREADS, 0, st>>>(run_flag, N, cnt.p);
  KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt.p, off.p, (int)(ntile + 1), st);
  }));
  k_flag_write<<<(unsigned)ntile, CF_THREADS, 0, st>>>(run_flag, N, off.p, rl.run_start.p);
  KCUDA(ctx, cudaMemcpyAsync(rl.m_dev.p, off.p + ntile, 4, cudaMemcpyDeviceToDevice, st));
  return KARETO_OK;
}

// With M (read by the caller): per run its request, length and first previous position.
kareto_status run_list_finish(kareto_ctx *ctx, uint64_t N, const uint32_t *prev_c, const uint32_t *req,
                              uint32_t req_base, const uint32_t *s, uint32_t pos_base, int M, RunList &rl) {
  rl.M = M;
  if (M == 0) return KARETO_OK;
  KTRY(rl.run_req.alloc(ctx, M)); KTRY(rl.run_len.alloc(ctx, M)); KTRY(rl.run_p0.alloc(ctx, M));
  Pass ps(ctx, "K3_run_info", 1, 1);
  k_run_info<<<grid_for(M, 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(rl.run_start.p, rl.m_dev.p, N, req, req_base,
                                                                         s, pos_base, prev_c, rl.run_req.p,
                                                                         rl.run_len.p, rl.run_p0.p);
  return KARETO_OK;
}

// K3 over n accesses (local positions 0..n-1) whose previous positions prev_c are given in
// coordinates [0, y_range) where local position i sits at y_off + i (whole trace: y_off = 0,
// y_range = n; a time shard prepends its boundary LRU stack, trace_shard.cu).
kareto_status stack_depth(kareto_ctx *ctx, uint64_t N, uint64_t y_range, const uint32_t *prev_c,
                          const uint32_t *req, uint32_t req_base, const uint32_t *s, uint32_t pos_base,
                          uint32_t y_off, const uint8_t *run_flag, uint32_t *depth, int64_t *n_runs,
                          uint4 **runs_out) {
  *n_runs = 0;
  if (N == 0) return KARETO_OK;
  RunList rl;
  KTRY(run_list_start(ctx, N, run_flag, rl));
  int M = 0;
  KCUDA(ctx, cudaMemcpyAsync(&M, rl.m_dev.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  KCUDA(ctx, cudaStreamSynchronize(ctx->stream));
  KTRY(run_list_finish(ctx, N, prev_c, req, req_base, s, pos_base, M, rl));
  return stack_depth_runs(ctx, N, y_range, s, pos_base, y_off, rl, depth, n_runs, runs_out);
}

// K3 proper over a run list (run_list_start / _finish).
kareto_status stack_depth_runs(kareto_ctx *ctx, uint64_t N, uint64_t y_range, const uint32_t *s,
                               uint32_t pos_base, uint32_t y_off, RunList &rl, uint32_t *depth, int64_t *n_runs,
                               uint4 **runs_out) {
  *n_runs = 0;
  if (N == 0) return KARETO_OK;
  if (y_range >= (1ull << 31)) return fail(ctx, KARETO_E_OVERFLOW, "stack depth pass supports < 2^31 positions");
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  if (depth) KCUDA(ctx, cudaMemsetAsync(depth, 0xFF, 4 * N, st));  // first accesses: UINT32_MAX
  DBuf<uint8_t> tmp;
  const int M = rl.M;
  *n_runs = M;
  if (M == 0) return KARETO_OK;
  DBuf<uint32_t> &run_start = rl.run_start, &run_req = rl.run_req, &run_len = rl.run_len, &run_p0 = rl.run_p0;
  DBuf<int> &m_dev = rl.m_dev;
  if (runs_out) KMALLOC(ctx, *runs_out, sizeof(uint4) * (size_t)M, st);
  const uint64_t NI = 2ull * (uint64_t)M;  // items
  DBuf<uint2> buf[2];
  KTRY(buf[0].alloc(ctx, NI)); KTRY(buf[1].alloc(ctx, NI));
  {
    Pass ps(ctx, "K3_run_items", 1, 1);
    k_run_items<<<grid_for(M, 256, 8 * sms), 256, 0, st>>>(m_dev.p, run_req.p, run_len.p, run_p0.p, buf[0].p);
  }
  int B = 1;
  while ((1ull << B) < y_range) B++;
  const int LB = B < SD_LOCAL_BITS ? B : SD_LOCAL_BITS;
  const int H = B - LB;
  const int npass = (H + 7) / 8;
  DBuf<uint32_t> A;
  KTRY(A.alloc(ctx, y_range));
  DBuf<uint64_t> seg_start, seg_len;
  KTRY(seg_start.alloc(ctx, 1)); KTRY(seg_len.alloc(ctx, 1));
  k_single_segment<<<1, 1, 0, st>>>(m_dev.p, seg_start.p, seg_len.p);
  ctx->own_launches++;
  uint32_t nseg = 1;
  int cur = 0;
  int shift = B, consumed = 0;
  for (int p = 0; p < npass; p++) {
    int bits = (H - consumed + (npass - p) - 1) / (npass - p);  // spread H bits over the passes
    shift -= bits;
    consumed += bits;
    const int bins = 1 << bits;
    DBuf<Tile> tiles;
    DBuf<uint32_t> seg_tile0, seg_ntiles;
    KTRY(seg_tile0.alloc(ctx, nseg)); KTRY(seg_ntiles.alloc(ctx, nseg));
    uint32_t ntiles;
    {
      Pass ps(ctx, "K3_tiles", 1, 2);
      k_sd_tiles<<<grid_for(nseg, 256, 1024), 256, 0, st>>>(nseg, seg_len.p, nullptr, seg_ntiles.p, nullptr, 0);
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, seg_ntiles.p, seg_tile0.p, (int)nseg, st);
      }));
      // upper bound of the tile count (no host sync): every segment rounds up by < 1 tile
      ntiles = (uint32_t)((NI + SD_TILE - 1) / SD_TILE + nseg);
      KTRY(tiles.alloc(ctx, ntiles));
      KCUDA(ctx, cudaMemsetAsync(tiles.p, 0xFF, sizeof(Tile) * ntiles, st));
      k_sd_tiles<<<grid_for(nseg, 256, 1024), 256, 0, st>>>(nseg, seg_len.p, seg_tile0.p, nullptr, tiles.p, 1);
    }
    DBuf<uint32_t> hist_all, hist_pts, off_all, off_pts;
    DBuf<unsigned long long> seg_tot;
    DBuf<uint64_t> nstart;
    size_t nh = (size_t)ntiles * bins;
    KTRY(hist_all.alloc(ctx, nh)); KTRY(hist_pts.alloc(ctx, nh));
    KTRY(off_all.alloc(ctx, nh)); KTRY(off_pts.alloc(ctx, nh));
    KTRY(hist_all.zero()); KTRY(hist_pts.zero());
    KTRY(seg_tot.alloc(ctx, (size_t)nseg * bins)); KTRY(seg_tot.zero());
    KTRY(nstart.alloc(ctx, (size_t)nseg * bins));
    PassArgs a{};
    a.in = buf[cur].p;
    a.tiles = tiles.p;
    a.seg_start = seg_start.p;
    a.seg_len = seg_len.p;
    a.seg_tile0 = seg_tile0.p;
    a.seg_ntiles = seg_ntiles.p;
    a.shift = shift;
    a.bits = bits;
    a.hist_all = hist_all.p;
    a.hist_pts = hist_pts.p;
    a.seg_tot = seg_tot.p;
    a.out = buf[cur ^ 1].p;
    {
      Pass ps(ctx, "K3_upsweep", 1, 1);
      k_sd_upsweep<<<ntiles, SD_WARPS * 32, 0, st>>>(a);
    }
    {
      Pass ps(ctx, "K3_scans", 0, 3);
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, hist_all.p, off_all.p, (int64_t)nh, st);
      }));
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, hist_pts.p, off_pts.p, (int64_t)nh, st);
      }));
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, (const uint64_t *)seg_tot.p, nstart.p, (int)(nseg * bins), st);
      }));
    }
    a.off_all = off_all.p;
    a.off_pts = off_pts.p;
    {
      Pass ps(ctx, "K3_downsweep", 1, 1);
      k_sd_downsweep<<<ntiles, SD_WARPS * 32, 0, st>>>(a);
    }
    DBuf<uint64_t> nlen;
    KTRY(nlen.alloc(ctx, (size_t)nseg * bins));
    KCUDA(ctx, cudaMemcpyAsync(nlen.p, seg_tot.p, 8 * (size_t)nseg * bins, cudaMemcpyDeviceToDevice, st));
    seg_start = std::move(nstart);
    seg_len = std::move(nlen);
    nseg *= bins;
    cur ^= 1;
  }
  {
    Pass ps(ctx, "K3_local", 1, 1);
    unsigned g = (unsigned)((nseg + LOCAL_WARPS - 1) / LOCAL_WARPS);
    if (g > (unsigned)(64 * sms)) g = (unsigned)(64 * sms);
    switch (LB) {
#define SD_CASE(b) case b: k_sd_local<b><<<g, LOCAL_WARPS * 32, 0, st>>>(buf[cur].p, seg_start.p, seg_len.p, nseg, A.p); break;
      SD_CASE(1) SD_CASE(2) SD_CASE(3) SD_CASE(4) SD_CASE(5) SD_CASE(6) SD_CASE(7) SD_CASE(8) SD_CASE(9)
      SD_CASE(10) SD_CASE(11)
#undef SD_CASE
      default: return fail(ctx, KARETO_E_INVALID, "bad local bits %d", LB);
    }
  }
  {
    Pass ps(ctx, depth ? "K3_expand" : "K3_runs_out", 1, 1);
    k_run_expand<<<grid_for(M, 256, 16 * sms), 256, 0, st>>>(m_dev.p, run_start.p, run_req.p, run_len.p, run_p0.p, s,
                                                             pos_base - y_off, A.p, depth,
                                                             runs_out ? *runs_out : nullptr);
  }
  return KARETO_OK;
}

// Per-access depths of a whole trace from its kept runs (d_{j0+t} = d0 - t; first accesses
// UINT32_MAX), on first use: the bench step's K4 reads the runs only (eval.cu k_hist_runs).
__global__ void __launch_bounds__(256) k_runs_depth(int64_t M, const uint4 *__restrict__ runs,
                                                    uint32_t *__restrict__ depth) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; q0 < M; q0 += nw * 32) {
    const int64_t q = q0 + lane;
    const uint4 rn = q < M ? runs[q] : make_uint4(0, 0, 0, 0);
    const int nk = M - q0 < 32 ? (int)(M - q0) : 32;
    for (int k = 0; k < nk; k++) {
      const uint32_t jk = __shfl_sync(0xFFFFFFFFu, rn.x, k), Lk = __shfl_sync(0xFFFFFFFFu, rn.y, k);
      const uint32_t bk = __shfl_sync(0xFFFFFFFFu, rn.z, k);
      for (uint32_t t = lane; t < Lk; t += 32) depth[jk + t] = bk - t;
    }
  }
}

kareto_status ensure_depth(kareto_ctx *ctx, kareto_trace *tr) {
  if (tr->depth_ready) return KARETO_OK;
  cudaStream_t st = ctx->stream;
  const uint64_t n = (uint64_t)(tr->pos_hi - tr->pos_lo);
  if (n > 0) {
    Pass ps(ctx, "K3_depth", 1, 1);
    KCUDA(ctx, cudaMemsetAsync(tr->depth, 0xFF, 4 * n, st));
    if (tr->n_runs > 0)
      k_runs_depth<<<grid_for(tr->n_runs, 256, 16 * ctx->num_sms), 256, 0, st>>>(tr->n_runs, tr->runs, tr->depth);
  }
  tr->depth_ready = true;
  return KARETO_OK;
}

}  // namespace kareto

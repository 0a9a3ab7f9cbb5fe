// stack_depth.cu -- row a4, K3: exact LRU stack depth of every reuse access.
//
// The pre-request LRU depth of access j of request r with previous access p is
//     d_j = s_r - p - A_j,   A_j = #{ i < s_r : prev[i] >= p }
// (live positions in [p, s_r); the O2 oracle computes the same
// with a sequential Fenwick tree).  A_j is an offline 2-D dominance count.  Here it is
// computed by an MSD radix partition *with counting*: the stream of items
//     for each request r in order:  queries (y = prev[j]) of its reuse accesses,
//                                    then points (y = prev[j]) of its reuse accesses
// (array order = time order x) is stably partitioned by the high digits of y; at every
// level a query adds the number of EARLIER points of its segment whose digit is larger
// (those have y > y_q), and the segment with equal digit recurses.  Two 8-bit global
// passes (for N <= 2^27) leave segments of 2048 consecutive y values, which one warp
// finishes with a 2048-bit shared-memory bitmap.  Equal y only occurs for a query and
// its own point, which comes later, so "y > y_q" == "prev >= p".
//
// Item = uint2 {y, w}: w = running count for a query, 0xFFFFFFFF for a point.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace kareto {

constexpr int SD_WARPS = 8;
constexpr int SD_CHUNKS = 16;                          // chunks of 32 items per warp per tile
constexpr int SD_TILE = SD_WARPS * SD_CHUNKS * 32;     // 4096 items per tile
constexpr int SD_LOCAL_BITS = 11;
constexpr uint32_t kPoint = 0xFFFFFFFFu;

struct VirtualIn {  // pass-1 input generated on the fly from prev[] / req[] / s[]
  const uint32_t *req, *s, *prev;
  uint64_t M;       // 2N virtual items
};

__device__ __forceinline__ bool virtual_item(const VirtualIn &vin, uint64_t v, uint2 &it) {
  uint32_t r = vin.req[v >> 1];
  uint32_t sr = vin.s[r], n = vin.s[r + 1] - sr;
  uint32_t off = (uint32_t)(v - 2 * (uint64_t)sr);
  bool q = off < n;
  uint32_t j = sr + (q ? off : off - n);
  uint32_t p = vin.prev[j];
  it = make_uint2(p, q ? 0u : kPoint);
  return p != kNone;
}

struct Tile {
  uint32_t seg, t;   // segment, local tile index
};

struct PassArgs {
  // input
  const uint2 *in;       // nullptr => virtual input
  VirtualIn vin;
  const Tile *tiles;     // per CTA tile descriptor (nullptr for virtual: seg 0, t = blockIdx)
  const uint64_t *seg_start;   // [nseg] start offsets of segments in `in`
  const uint64_t *seg_len;     // [nseg]
  const uint32_t *seg_tile0;   // [nseg] first global tile of the segment
  const uint32_t *seg_ntiles;  // [nseg]
  uint32_t n_tiles_virtual;
  int shift, bits;       // digit = (y >> shift) & (2^bits - 1)
  // outputs
  uint32_t *hist_all, *hist_pts;     // [tiles * bins] layout tile0*bins + d*ntiles + t
  unsigned long long *seg_tot;       // [nseg * bins] (upsweep)
  const uint32_t *off_all, *off_pts; // exclusive sums of the two histograms (downsweep)
  uint2 *out;
};

__device__ __forceinline__ void tile_geometry(const PassArgs &a, uint32_t bid, uint32_t &seg, uint32_t &t,
                                              uint64_t &beg, uint64_t &end, uint32_t &tile0, uint32_t &ntiles) {
  if (a.in == nullptr) {
    seg = 0; t = bid; tile0 = 0; ntiles = a.n_tiles_virtual;
    beg = (uint64_t)bid * SD_TILE;
    end = beg + SD_TILE < a.vin.M ? beg + SD_TILE : a.vin.M;
  } else {
    Tile td = a.tiles[bid];
    seg = td.seg; t = td.t;
    tile0 = a.seg_tile0[seg]; ntiles = a.seg_ntiles[seg];
    uint64_t s0 = a.seg_start[seg], L = a.seg_len[seg];
    beg = s0 + (uint64_t)t * SD_TILE;
    uint64_t e = s0 + (uint64_t)(t + 1) * SD_TILE;
    end = e < s0 + L ? e : s0 + L;
  }
}

__device__ __forceinline__ bool load_item(const PassArgs &a, uint64_t i, uint2 &it) {
  if (a.in == nullptr) return virtual_item(a.vin, i, it);
  it = a.in[i];
  return true;
}

// ---- upsweep: per-tile digit histograms (all items, points) + segment totals
__global__ void __launch_bounds__(SD_WARPS * 32) k_sd_upsweep(PassArgs a) {
  __shared__ uint32_t h_all[256], h_pts[256];
  const int bins = 1 << a.bits;
  for (int i = threadIdx.x; i < bins; i += blockDim.x) { h_all[i] = 0; h_pts[i] = 0; }
  __syncthreads();
  uint32_t seg, t, tile0, ntiles;
  uint64_t beg, end;
  tile_geometry(a, blockIdx.x, seg, t, beg, end, tile0, ntiles);
  for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    uint2 it;
    if (!load_item(a, i, it)) continue;
    uint32_t d = (it.x >> a.shift) & (bins - 1);
    atomicAdd(&h_all[d], 1u);
    if (it.y == kPoint) atomicAdd(&h_pts[d], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += blockDim.x) {
    size_t idx = (size_t)tile0 * bins + (size_t)d * ntiles + t;
    a.hist_all[idx] = h_all[d];
    a.hist_pts[idx] = h_pts[d];
    if (h_all[d]) atomicAdd(&a.seg_tot[(size_t)seg * bins + d], (unsigned long long)h_all[d]);
  }
}

// ---- downsweep: stable scatter by digit + query contributions
__global__ void __launch_bounds__(SD_WARPS * 32) k_sd_downsweep(PassArgs a) {
  __shared__ uint32_t run_all[SD_WARPS][256];
  __shared__ uint32_t run_pts[SD_WARPS][256];
  __shared__ uint32_t suf[SD_WARPS][256];
  const int bins = 1 << a.bits;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t seg, t, tile0, ntiles;
  uint64_t beg, end;
  tile_geometry(a, blockIdx.x, seg, t, beg, end, tile0, ntiles);
  const uint64_t wbeg = beg + (uint64_t)wid * SD_CHUNKS * 32;
  // phase A: per-warp histograms of this warp's contiguous sub-range
  for (int d = lane; d < bins; d += 32) { run_all[wid][d] = 0; run_pts[wid][d] = 0; }
  __syncwarp();
  for (int c = 0; c < SD_CHUNKS; c++) {
    uint64_t i = wbeg + (uint64_t)c * 32 + lane;
    uint2 it;
    bool live = i < end && load_item(a, i, it);
    if (live) {
      uint32_t d = (it.x >> a.shift) & (bins - 1);
      atomicAdd(&run_all[wid][d], 1u);
      if (it.y == kPoint) atomicAdd(&run_pts[wid][d], 1u);
    }
  }
  __syncthreads();
  // phase B: running offsets at the start of each warp's sub-range
  for (int d = threadIdx.x; d < bins; d += blockDim.x) {
    size_t idx = (size_t)tile0 * bins + (size_t)d * ntiles + t;
    size_t idx0 = (size_t)tile0 * bins + (size_t)d * ntiles;
    uint32_t ra = a.off_all[idx];
    uint32_t rp = a.off_pts[idx] - a.off_pts[idx0];  // points of digit d in earlier tiles of the segment
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
    // suffix sums over digits of the running point counts: suf[d] = sum_{d' > d} run_pts[d']
    {
      uint32_t v[8], tot = 0;
      int per = bins > 32 ? bins / 32 : 1;
      int base = lane * per;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        v[k] = (k < per && base + k < bins) ? run_pts[wid][base + k] : 0u;
        tot += v[k];
      }
      // exclusive suffix over lanes: sum of totals of higher lanes
      uint32_t incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t o = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += o;
      }
      uint32_t acc = incl - tot;  // higher lanes
#pragma unroll
      for (int k = 7; k >= 0; k--) {
        if (k < per && base + k < bins) suf[wid][base + k] = acc;
        acc += v[k];
      }
    }
    __syncwarp();
    uint64_t i = wbeg + (uint64_t)c * 32 + lane;
    uint2 it = make_uint2(0, 0);
    bool live = i < end && load_item(a, i, it);
    bool isp = live && it.y == kPoint;
    uint32_t d = live ? (it.x >> a.shift) & (bins - 1) : 0u;
    // earlier lanes that are points with a larger digit (bit-plane ballots)
    unsigned gt = 0, eq = __ballot_sync(0xffffffffu, isp);
    for (int b = a.bits - 1; b >= 0; b--) {
      unsigned pb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      if (!((d >> b) & 1u)) gt |= eq & pb;
      eq &= ((d >> b) & 1u) ? pb : ~pb;
    }
    unsigned lm = __ballot_sync(0xffffffffu, live);
    unsigned ptsm = __ballot_sync(0xffffffffu, isp);
    unsigned same = __match_any_sync(0xffffffffu, live ? d : 0xFFFFFFFFu);
    if (live) {
      uint32_t pos = run_all[wid][d] + __popc(same & lm & lt);
      uint2 o = it;
      if (!isp) o.y = it.y + suf[wid][d] + __popc(gt & lt);
      a.out[pos] = o;
    }
    __syncwarp();
    // advance running counts (leader of each digit group)
    if (live && (__ffs(same & lm) - 1) == lane) {
      run_all[wid][d] += __popc(same & lm);
      run_pts[wid][d] += __popc(same & ptsm);
    }
    __syncwarp();
  }
}

// ---- local pass: one warp per segment of 2^LB consecutive y values (bitmap in smem)
template <int LB>
__global__ void __launch_bounds__(256) k_sd_local(const uint2 *__restrict__ in, VirtualIn vin,
                                                  const uint64_t *__restrict__ seg_start,
                                                  const uint64_t *__restrict__ seg_len, uint32_t nseg,
                                                  uint32_t *__restrict__ A) {
  constexpr int W = (1 << LB) / 32 > 0 ? (1 << LB) / 32 : 1;  // bitmap words
  __shared__ uint32_t bm[8][W];
  __shared__ uint32_t sufw[8][W];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t seg = blockIdx.x * 8 + wid; seg < nseg; seg += gridDim.x * 8) {
    uint64_t s0, L;
    if (in) { s0 = seg_start[seg]; L = seg_len[seg]; }
    else { s0 = 0; L = vin.M; }
    if (L == 0) continue;
    for (int w = lane; w < W; w += 32) { bm[wid][w] = 0; sufw[wid][w] = 0; }
    __syncwarp();
    for (uint64_t c0 = 0; c0 < L; c0 += 32) {
      uint64_t i = s0 + c0 + lane;
      uint2 it = make_uint2(0, 0);
      bool live = c0 + lane < L;
      if (live) {
        if (in) it = in[i];
        else live = virtual_item(vin, i, it);
      }
      bool isp = live && it.y == kPoint;
      uint32_t yl = it.x & ((1u << LB) - 1u);
      unsigned gt = 0, eq = __ballot_sync(0xffffffffu, isp);
#pragma unroll
      for (int b = LB - 1; b >= 0; b--) {
        unsigned pb = __ballot_sync(0xffffffffu, (yl >> b) & 1u);
        if (!((yl >> b) & 1u)) gt |= eq & pb;
        eq &= ((yl >> b) & 1u) ? pb : ~pb;
      }
      if (live && !isp) {
        uint32_t wq = yl >> 5, bq = yl & 31;
        uint32_t above = (bq == 31) ? 0u : (bm[wid][wq] >> (bq + 1));
        uint32_t cnt = sufw[wid][wq] + __popc(above) + __popc(gt & lt);
        A[it.x] = it.y + cnt;
      }
      __syncwarp();
      if (isp) atomicOr(&bm[wid][yl >> 5], 1u << (yl & 31));
      __syncwarp();
      // suffix popcounts over bitmap words: sufw[w] = sum_{w' > w} popc(bm[w'])
      if (W <= 32) {
        uint32_t pc = lane < W ? __popc(bm[wid][lane]) : 0u;
        uint32_t incl = pc;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t o = __shfl_down_sync(0xffffffffu, incl, off);
          if (lane + off < 32) incl += o;
        }
        if (lane < W) sufw[wid][lane] = incl - pc;
      } else {
        constexpr int PER = W / 32;
        uint32_t pc[PER > 0 ? PER : 1], tot = 0;
#pragma unroll
        for (int k = 0; k < PER; k++) { pc[k] = __popc(bm[wid][lane * PER + k]); tot += pc[k]; }
        uint32_t incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          uint32_t o = __shfl_down_sync(0xffffffffu, incl, off);
          if (lane + off < 32) incl += o;
        }
        uint32_t acc = incl - tot;
#pragma unroll
        for (int k = PER - 1; k >= 0; k--) { sufw[wid][lane * PER + k] = acc; acc += pc[k]; }
      }
      __syncwarp();
    }
  }
}

// d_j = s_r - p - A[p]  (UINT32_MAX for first accesses)
__global__ void k_sd_finalize(uint64_t N, const uint32_t *__restrict__ prev, const uint32_t *__restrict__ req,
                              const uint32_t *__restrict__ s, const uint32_t *__restrict__ A,
                              uint32_t *__restrict__ depth) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t p = prev[j];
    depth[j] = p == kNone ? kNone : s[req[j]] - p - A[p];
  }
}

__global__ void k_sd_tiles(uint32_t nseg, const uint64_t *__restrict__ seg_len, const uint32_t *__restrict__ tile0,
                           uint32_t *__restrict__ ntiles_out, Tile *__restrict__ tiles, int write) {
  for (uint32_t sgi = blockIdx.x * blockDim.x + threadIdx.x; sgi < nseg; sgi += gridDim.x * blockDim.x) {
    uint32_t nt = (uint32_t)((seg_len[sgi] + SD_TILE - 1) / SD_TILE);
    if (!write) { ntiles_out[sgi] = nt; continue; }
    for (uint32_t t = 0; t < nt; t++) tiles[tile0[sgi] + t] = Tile{sgi, t};
  }
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

kareto_status stack_depth(kareto_ctx *ctx, kareto_trace *tr) {
  const uint64_t N = (uint64_t)tr->N;
  if (N == 0) return KARETO_OK;
  if (N >= (1ull << 31)) return fail(ctx, KARETO_E_OVERFLOW, "stack depth pass supports < 2^31 accesses");
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  int B = 1;
  while ((1ull << B) < N) B++;
  const int LB = B < SD_LOCAL_BITS ? B : SD_LOCAL_BITS;
  const int H = B - LB;
  const int npass = (H + 7) / 8;
  VirtualIn vin{tr->req, tr->s, tr->prev, 2 * N};
  DBuf<uint32_t> A;
  KTRY(A.alloc(ctx, N));
  DBuf<uint8_t> tmp;
  DBuf<uint2> buf[2];
  DBuf<uint64_t> seg_start, seg_len;  // segments of the current input
  uint32_t nseg = 1;
  const uint2 *cur = nullptr;         // nullptr => virtual
  int shift = B;
  int consumed = 0;
  if (npass > 0) {
    KTRY(buf[0].alloc(ctx, 2 * N));
    KTRY(buf[1].alloc(ctx, 2 * N));
  }
  for (int p = 0; p < npass; p++) {
    int bits = (H - consumed + (npass - p) - 1) / (npass - p);  // spread H bits over the passes
    shift -= bits;
    consumed += bits;
    const int bins = 1 << bits;
    // tile descriptors
    uint32_t ntiles;
    DBuf<Tile> tiles;
    DBuf<uint32_t> seg_tile0, seg_ntiles;
    KTRY(seg_tile0.alloc(ctx, nseg)); KTRY(seg_ntiles.alloc(ctx, nseg));
    if (cur == nullptr) {
      ntiles = (uint32_t)((vin.M + SD_TILE - 1) / SD_TILE);
    } else {
      Pass ps(ctx, "K3_tiles", 1, 2);
      k_sd_tiles<<<grid_for(nseg, 256, 1024), 256, 0, st>>>(nseg, seg_len.p, nullptr, seg_ntiles.p, nullptr, 0);
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, seg_ntiles.p, seg_tile0.p, (int)nseg, st);
      }));
      uint32_t last0 = 0, lastn = 0;
      KCUDA(ctx, cudaMemcpyAsync(&last0, seg_tile0.p + nseg - 1, 4, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaMemcpyAsync(&lastn, seg_ntiles.p + nseg - 1, 4, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      ntiles = last0 + lastn;
      KTRY(tiles.alloc(ctx, ntiles ? ntiles : 1));
      k_sd_tiles<<<grid_for(nseg, 256, 1024), 256, 0, st>>>(nseg, seg_len.p, seg_tile0.p, nullptr, tiles.p, 1);
    }
    DBuf<uint32_t> hist_all, hist_pts, off_all, off_pts;
    DBuf<unsigned long long> seg_tot;
    DBuf<uint64_t> nstart;
    size_t nh = (size_t)ntiles * bins;
    KTRY(hist_all.alloc(ctx, nh)); KTRY(hist_pts.alloc(ctx, nh));
    KTRY(off_all.alloc(ctx, nh)); KTRY(off_pts.alloc(ctx, nh));
    KTRY(seg_tot.alloc(ctx, (size_t)nseg * bins)); KTRY(seg_tot.zero());
    KTRY(nstart.alloc(ctx, (size_t)nseg * bins));
    PassArgs a{};
    a.in = cur;
    a.vin = vin;
    a.tiles = tiles.p;
    a.seg_start = seg_start.p;
    a.seg_len = seg_len.p;
    a.seg_tile0 = seg_tile0.p;
    a.seg_ntiles = seg_ntiles.p;
    a.n_tiles_virtual = ntiles;
    a.shift = shift;
    a.bits = bits;
    a.hist_all = hist_all.p;
    a.hist_pts = hist_pts.p;
    a.seg_tot = seg_tot.p;
    a.out = buf[p & 1].p;
    if (ntiles > 0) {
      Pass ps(ctx, p == 0 ? "K3_upsweep1" : "K3_upsweep2", 1, 1);
      k_sd_upsweep<<<ntiles, SD_WARPS * 32, 0, st>>>(a);
    }
    if (nh > 0) {
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
    if (ntiles > 0) {
      Pass ps(ctx, p == 0 ? "K3_downsweep1" : "K3_downsweep2", 1, 1);
      k_sd_downsweep<<<ntiles, SD_WARPS * 32, 0, st>>>(a);
    }
    // next segments: (old segment, digit), starts = exclusive sums of seg_tot
    DBuf<uint64_t> nlen;
    KTRY(nlen.alloc(ctx, (size_t)nseg * bins));
    KCUDA(ctx, cudaMemcpyAsync(nlen.p, seg_tot.p, 8 * (size_t)nseg * bins, cudaMemcpyDeviceToDevice, st));
    seg_start = std::move(nstart);
    seg_len = std::move(nlen);
    nseg *= bins;
    cur = buf[p & 1].p;
  }
  {
    Pass ps(ctx, "K3_local", 1, 1);
    unsigned g = (unsigned)((nseg + 7) / 8);
    if (g > (unsigned)(64 * sms)) g = (unsigned)(64 * sms);
    switch (LB) {
#define SD_CASE(b) case b: k_sd_local<b><<<g, 256, 0, st>>>(cur, vin, seg_start.p, seg_len.p, nseg, A.p); break;
      SD_CASE(1) SD_CASE(2) SD_CASE(3) SD_CASE(4) SD_CASE(5) SD_CASE(6) SD_CASE(7) SD_CASE(8) SD_CASE(9)
      SD_CASE(10) SD_CASE(11)
#undef SD_CASE
      default: return fail(ctx, KARETO_E_INVALID, "bad local bits %d", LB);
    }
  }
  {
    Pass ps(ctx, "K3_finalize", 1, 1);
    k_sd_finalize<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->prev, tr->req, tr->s, A.p, tr->depth);
  }
  return KARETO_OK;
}

}  // namespace kareto

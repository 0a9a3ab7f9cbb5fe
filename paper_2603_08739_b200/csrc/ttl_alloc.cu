// ttl_alloc.cu -- row f2: Alg. 2 "ROI-Aware TTL Allocation" over the exact
// group curves of P:750-752:
//     H_g(t) = #{delta in Delta_g : delta <= t},   C_g(t) = |B_g| t + sum min(t, delta).
//
// B200 design.  The curves are built once per call from the trace resident in HBM: every
// non-first access contributes the key (g << 32 | delta); one CUB radix sort + run-length
// encode gives each group's distinct intervals with their counts, two CUB scans give the
// cumulative H and sum(delta) per distinct interval (the jump table).  Everything Alg. 2 asks
// of the curves is then data-parallel over jump points:
//   * ROI argmax per group (l.4-5, R43): one CTA per group, exact u128 cross-multiplied compare;
//   * the local solve from each start (l.15, R44): each step is one launch in which a CTA per
//     group finds its best up- (or down-) move over all its jump points, exact in u128; the host
//     takes the best group (K+1 values) and applies it;
//   * batched Sum H / Sum C of TTL vectors (kareto_ttl_eval): thread per (vector, group) binary
//     search; the same kernel probes 64 uniform TTLs per round for the R54 start (the largest
//     uniform TTL within the budget, R54).
// The decisions are integer-exact, so the result equals the oracle's (oracle/ttl_alloc.py).
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "internal.cuh"

namespace kareto {

typedef unsigned __int128 u128;
constexpr uint32_t TTL_MAX_MS = 0xFFFFFFFEu;

// ------------------------------------------------------------------ curve tables
struct Curves {
  int G = 0;
  DBuf<uint32_t> v;         // [m] distinct interval (ms) of each jump row, rows grouped by g
  DBuf<uint64_t> H, S;      // [m] cumulative count / sum of intervals within the group (incl. row)
  DBuf<int64_t> gfirst, gend;  // [G] first row with v > 0, end row
  DBuf<uint64_t> h0, Ug, Ng;   // [G] H(0), |B_g|, N_g
  std::vector<int64_t> hfirst, hend;
  std::vector<uint64_t> hh0, hU, hN;
};

__global__ void k_reuse_keys(uint64_t N, const uint32_t *__restrict__ delta, const uint32_t *__restrict__ req,
                             const uint16_t *__restrict__ grp, int G, uint64_t *__restrict__ key) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = delta[j];
    key[j] = d == kNone ? ((uint64_t)G << 32) : (((uint64_t)grp[req[j]] << 32) | d);
  }
}

__global__ void k_run_fields(const uint64_t *__restrict__ ukey, const uint32_t *__restrict__ cnt,
                             const int *__restrict__ m_ptr, int G, uint32_t *__restrict__ v,
                             uint64_t *__restrict__ c64, uint64_t *__restrict__ vc) {
  const int m = *m_ptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const uint64_t k = ukey[i];
    const bool real = (int)(k >> 32) < G;
    v[i] = (uint32_t)k;
    c64[i] = real ? cnt[i] : 0;
    vc[i] = real ? (uint64_t)(uint32_t)k * cnt[i] : 0;
  }
}

// group ranges and per-group rebasing of the global inclusive scans
__global__ void k_group_bounds(const uint64_t *__restrict__ ukey, const int *__restrict__ m_ptr, int G,
                               int64_t *__restrict__ gstart, int64_t *__restrict__ gend) {
  const int m = *m_ptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int g = (int)(ukey[i] >> 32);
    if (g >= G) continue;
    if (i == 0 || (int)(ukey[i - 1] >> 32) != g) gstart[g] = i;
    if (i == m - 1 || (int)(ukey[i + 1] >> 32) != g) gend[g] = i + 1;
  }
}

__global__ void k_rebase(const uint64_t *__restrict__ ukey, const int *__restrict__ m_ptr, int G,
                         const int64_t *__restrict__ gstart, const uint64_t *__restrict__ Hg,
                         const uint64_t *__restrict__ Sg, uint64_t *__restrict__ H, uint64_t *__restrict__ S) {
  const int m = *m_ptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int g = (int)(ukey[i] >> 32);
    if (g >= G) continue;
    const int64_t s0 = gstart[g];
    H[i] = Hg[i] - (s0 > 0 ? Hg[s0 - 1] : 0);
    S[i] = Sg[i] - (s0 > 0 ? Sg[s0 - 1] : 0);
  }
}

__global__ void k_group_meta(int G, const int64_t *__restrict__ gstart, int64_t *__restrict__ gend,
                             const uint32_t *__restrict__ v, const uint64_t *__restrict__ H,
                             int64_t *__restrict__ gfirst, uint64_t *__restrict__ h0) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int64_t s = gstart[g], e = gend[g];
  if (e <= s) {  // empty group
    gfirst[g] = s;
    gend[g] = s;
    h0[g] = 0;
    return;
  }
  const bool zero = v[s] == 0;
  gfirst[g] = zero ? s + 1 : s;
  h0[g] = zero ? H[s] : 0;
}

template <typename F>
static kareto_status cub_do(kareto_ctx *ctx, DBuf<uint8_t> &tmp, F &&f) {
  size_t bytes = 0;
  KCUDA(ctx, f((void *)nullptr, bytes));
  if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
  size_t b2 = tmp.n;
  KCUDA(ctx, f((void *)tmp.p, b2));
  return KARETO_OK;
}

static kareto_status build_curves(kareto_ctx *ctx, const kareto_trace *tr, Curves &cv) {
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int G = tr->K + 1;
  const uint64_t N = (uint64_t)tr->N;
  cv.G = G;
  DBuf<uint8_t> tmp;
  KTRY(cv.gfirst.alloc(ctx, G)); KTRY(cv.gend.alloc(ctx, G)); KTRY(cv.h0.alloc(ctx, G));
  KTRY(cv.Ug.alloc(ctx, G)); KTRY(cv.Ng.alloc(ctx, G));
  DBuf<int64_t> gstart;
  KTRY(gstart.alloc(ctx, G));
  KCUDA(ctx, cudaMemsetAsync(gstart.p, 0, 8 * G, st));
  KCUDA(ctx, cudaMemsetAsync(cv.gend.p, 0, 8 * G, st));
  int m = 0;
  if (N > 0) {
    Pass ps(ctx, "F2_curves", 1, 5);
    DBuf<uint64_t> key, keys, ukey, c64, vc, Hg, Sg;
    DBuf<uint32_t> cnt;
    DBuf<int> m_dev;
    KTRY(key.alloc(ctx, N)); KTRY(keys.alloc(ctx, N)); KTRY(m_dev.alloc(ctx, 1));
    k_reuse_keys<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->delta, tr->req, tr->grp, G, key.p);
    int gb = 1;
    while ((1 << gb) <= G) gb++;
    KTRY(cub_do(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortKeys(t, b, key.p, keys.p, (int64_t)N, 0, 32 + gb, st);
    }));
    key.release();
    KTRY(ukey.alloc(ctx, N)); KTRY(cnt.alloc(ctx, N));
    KTRY(cub_do(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRunLengthEncode::Encode(t, b, keys.p, ukey.p, cnt.p, m_dev.p, (int64_t)N, st);
    }));
    keys.release();
    KCUDA(ctx, cudaMemcpyAsync(&m, m_dev.p, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    KTRY(cv.v.alloc(ctx, m)); KTRY(c64.alloc(ctx, m)); KTRY(vc.alloc(ctx, m)); KTRY(Hg.alloc(ctx, m));
    KTRY(Sg.alloc(ctx, m)); KTRY(cv.H.alloc(ctx, m)); KTRY(cv.S.alloc(ctx, m));
    k_run_fields<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(ukey.p, cnt.p, m_dev.p, G, cv.v.p, c64.p, vc.p);
    KTRY(cub_do(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceScan::InclusiveSum(t, b, c64.p, Hg.p, m, st); }));
    KTRY(cub_do(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceScan::InclusiveSum(t, b, vc.p, Sg.p, m, st); }));
    k_group_bounds<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(ukey.p, m_dev.p, G, gstart.p, cv.gend.p);
    k_rebase<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(ukey.p, m_dev.p, G, gstart.p, Hg.p, Sg.p, cv.H.p, cv.S.p);
    k_group_meta<<<grid_for(G, 128), 128, 0, st>>>(G, gstart.p, cv.gend.p, cv.v.p, cv.H.p, cv.gfirst.p, cv.h0.p);
  } else {
    KTRY(cv.v.alloc(ctx, 1)); KTRY(cv.H.alloc(ctx, 1)); KTRY(cv.S.alloc(ctx, 1));
    KCUDA(ctx, cudaMemsetAsync(cv.gfirst.p, 0, 8 * G, st));
    KCUDA(ctx, cudaMemsetAsync(cv.h0.p, 0, 8 * G, st));
  }
  cv.hU.resize(G);
  cv.hN.resize(G);
  for (int g = 0; g < G; g++) {
    cv.hU[g] = (uint64_t)tr->U_g[g];
    cv.hN[g] = (uint64_t)tr->reuse_g[g];
  }
  KCUDA(ctx, cudaMemcpyAsync(cv.Ug.p, cv.hU.data(), 8 * G, cudaMemcpyHostToDevice, st));
  KCUDA(ctx, cudaMemcpyAsync(cv.Ng.p, cv.hN.data(), 8 * G, cudaMemcpyHostToDevice, st));
  cv.hfirst.resize(G);
  cv.hend.resize(G);
  cv.hh0.resize(G);
  KCUDA(ctx, cudaMemcpyAsync(cv.hfirst.data(), cv.gfirst.p, 8 * G, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaMemcpyAsync(cv.hend.data(), cv.gend.p, 8 * G, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaMemcpyAsync(cv.hh0.data(), cv.h0.p, 8 * G, cudaMemcpyDeviceToHost, st));
  return sync(ctx, "ttl curves");
}

// C_g at a jump row (v, H, S): |B| v + S + v (N - H)
__device__ __forceinline__ uint64_t c_at(uint64_t U, uint64_t Ng, uint32_t v, uint64_t H, uint64_t S) {
  return U * v + S + (uint64_t)v * (Ng - H);
}

// (H, C) of group g at TTL t: the last jump row with v <= t
__device__ __forceinline__ void eval_at(const Curves *, const uint32_t *__restrict__ v, const uint64_t *__restrict__ H,
                                        const uint64_t *__restrict__ S, int64_t lo, int64_t hi, uint64_t h0,
                                        uint64_t U, uint64_t Ng, uint32_t t, uint64_t &h, uint64_t &c, int64_t &row) {
  int64_t a = lo, b = hi;  // first row with v > t
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (v[mid] <= t) a = mid + 1; else b = mid;
  }
  row = a - 1;  // lo - 1: the t = 0 point
  const uint64_t hh = a > lo ? H[a - 1] : h0;
  const uint64_t ss = a > lo ? S[a - 1] : 0;
  h = hh;
  c = U * t + ss + (uint64_t)t * (Ng - hh);
}

struct CurveView {
  const uint32_t *v;
  const uint64_t *H, *S;
  const int64_t *gfirst, *gend;
  const uint64_t *h0, *U, *N;
};

// ------------------------------------------------------------------ ROI (Alg. 2 l.4-5, R43)
struct Best {
  uint64_t h, c;
  int64_t row;
  uint32_t t;
  int valid;
};

__global__ void __launch_bounds__(256) k_roi(CurveView cv, int G, uint32_t *__restrict__ t_roi,
                                             uint64_t *__restrict__ h_roi, uint64_t *__restrict__ c_roi) {
  __shared__ uint64_t sh[256], sc[256];
  __shared__ uint32_t stt[256];
  __shared__ int sv[256];
  const int g = blockIdx.x;
  if (g >= G) return;
  const int64_t lo = cv.gfirst[g], hi = cv.gend[g];
  const uint64_t U = cv.U[g], Ng = cv.N[g], h0 = cv.h0[g];
  // candidate t = 1 (covers delta in {0, 1}) and every v >= 2
  uint64_t bh = 0, bc = 1;
  uint32_t bt = 0;
  int valid = 0;
  auto offer = [&](uint32_t t, uint64_t h, uint64_t c) {
    // larger h/c wins; ties -> smaller t
    if (!valid || (u128)h * bc > (u128)bh * c || ((u128)h * bc == (u128)bh * c && t < bt)) {
      bh = h; bc = c; bt = t; valid = 1;
    }
  };
  if (threadIdx.x == 0 && Ng > 0) {
    uint64_t h, c;
    int64_t row;
    eval_at(nullptr, cv.v, cv.H, cv.S, lo, hi, h0, U, Ng, 1u, h, c, row);
    if (c > 0) offer(1u, h, c);
  }
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t t = cv.v[i];
    if (t < 2) continue;
    offer(t, cv.H[i], c_at(U, Ng, t, cv.H[i], cv.S[i]));
  }
  sh[threadIdx.x] = bh; sc[threadIdx.x] = bc; stt[threadIdx.x] = bt; sv[threadIdx.x] = valid;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)blockDim.x; q++)
      if (sv[q]) {
        if (!valid || (u128)sh[q] * bc > (u128)bh * sc[q] || ((u128)sh[q] * bc == (u128)bh * sc[q] && stt[q] < bt)) {
          bh = sh[q]; bc = sc[q]; bt = stt[q]; valid = 1;
        }
      }
    t_roi[g] = valid ? bt : 0;
    h_roi[g] = valid ? bh : 0;
    c_roi[g] = valid ? bc : 0;
  }
}

// ------------------------------------------------------------------ batched evaluation
__global__ void k_ttl_eval(CurveView cv, int G, const uint32_t *__restrict__ ttl, int64_t n,
                           unsigned long long *__restrict__ hits, unsigned long long *__restrict__ cost) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n * G; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = x / G;
    const int g = (int)(x - q * G);
    uint64_t h, c;
    int64_t row;
    eval_at(nullptr, cv.v, cv.H, cv.S, cv.gfirst[g], cv.gend[g], cv.h0[g], cv.U[g], cv.N[g], ttl[x], h, c, row);
    atomicAdd(&hits[q], (unsigned long long)h);
    atomicAdd(&cost[q], (unsigned long long)c);
  }
}

// snap: per group the last jump row <= t (R44 (a))
__global__ void k_snap(CurveView cv, int G, const uint32_t *__restrict__ t, int64_t *__restrict__ row,
                       uint64_t *__restrict__ h, uint64_t *__restrict__ c) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  int64_t r;
  uint64_t hh, cc;
  const int64_t lo = cv.gfirst[g];
  eval_at(nullptr, cv.v, cv.H, cv.S, lo, cv.gend[g], cv.h0[g], cv.U[g], cv.N[g], t[g], hh, cc, r);
  // snapped to the jump point: its cost (not the cost at t)
  const uint32_t tj = r >= lo ? cv.v[r] : 0u;
  row[g] = r;
  h[g] = hh;
  c[g] = r >= lo ? c_at(cv.U[g], cv.N[g], tj, hh, cv.S[r]) : 0;
}

// best single-group move (R44 (b) down / (c) up) of every group; out: dh, dc, row (row = -2: none)
struct Move {
  uint64_t dh, dc;
  int64_t row;
};
__device__ __forceinline__ bool better_up(const Move &a, const Move &b) {  // a better than b?
  if (b.row == -2) return a.row != -2;
  if (a.row == -2) return false;
  const u128 l = (u128)a.dh * b.dc, r = (u128)b.dh * a.dc;
  return l > r || (l == r && a.row < b.row);
}
__device__ __forceinline__ bool better_down(const Move &a, const Move &b) {
  if (b.row == -2) return a.row != -2;
  if (a.row == -2) return false;
  const u128 l = (u128)a.dh * b.dc, r = (u128)b.dh * a.dc;
  return l < r || (l == r && a.row > b.row);
}

__global__ void __launch_bounds__(256) k_best_move(CurveView cv, int G, int up, const int64_t *__restrict__ pos,
                                                   const uint64_t *__restrict__ hc, const uint64_t *__restrict__ cc,
                                                   uint64_t rem, Move *__restrict__ out) {
  __shared__ Move sm[256];
  const int g = blockIdx.x;
  if (g >= G) return;
  const int64_t lo = cv.gfirst[g], hi = cv.gend[g], p = pos[g];
  const uint64_t U = cv.U[g], Ng = cv.N[g], H0 = hc[g], C0 = cc[g];
  Move best{0, 0, -2};
  if (up) {
    for (int64_t i = (p + 1 > lo ? p + 1 : lo) + threadIdx.x; i < hi; i += blockDim.x) {
      const uint64_t Hi = cv.H[i], Ci = c_at(U, Ng, cv.v[i], Hi, cv.S[i]);
      if (Ci <= C0 || Hi <= H0) continue;
      Move m{Hi - H0, Ci - C0, i};
      if (m.dc > rem) continue;
      if (better_up(m, best)) best = m;
    }
  } else {
    // the t = 0 point (row lo - 1): H = h0, C = 0
    if (threadIdx.x == 0 && p > lo - 1 && C0 > 0) {
      Move m{H0 - cv.h0[g], C0, lo - 1};
      best = m;
    }
    for (int64_t i = lo + threadIdx.x; i < p; i += blockDim.x) {
      const uint64_t Hi = cv.H[i], Ci = c_at(U, Ng, cv.v[i], Hi, cv.S[i]);
      if (C0 <= Ci) continue;
      Move m{H0 - Hi, C0 - Ci, i};
      if (better_down(m, best)) best = m;
    }
  }
  sm[threadIdx.x] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)blockDim.x; q++)
      if (up ? better_up(sm[q], best) : better_down(sm[q], best)) best = sm[q];
    out[g] = best;
  }
}

static CurveView view(const Curves &c) {
  return CurveView{c.v.p, c.H.p, c.S.p, c.gfirst.p, c.gend.p, c.h0.p, c.Ug.p, c.Ng.p};
}

static bool host_better(bool up, const Move &a, const Move &b) {
  if (b.row == -2) return a.row != -2;
  if (a.row == -2) return false;
  const u128 l = (u128)a.dh * b.dc, r = (u128)b.dh * a.dc;
  return up ? l > r : l < r;  // ties keep the earlier (smaller) group
}

// R44 local solve from t_start; returns the TTL vector and its totals
static kareto_status local_solve(kareto_ctx *ctx, const Curves &cv, const std::vector<uint32_t> &t_start, uint64_t B,
                                 std::vector<uint32_t> &t_out, uint64_t &hits, uint64_t &cost) {
  cudaStream_t st = ctx->stream;
  const int G = cv.G;
  DBuf<uint32_t> dt;
  DBuf<int64_t> dpos;
  DBuf<uint64_t> dh, dc;
  DBuf<Move> dmv;
  KTRY(dt.alloc(ctx, G)); KTRY(dpos.alloc(ctx, G)); KTRY(dh.alloc(ctx, G)); KTRY(dc.alloc(ctx, G));
  KTRY(dmv.alloc(ctx, G));
  KCUDA(ctx, cudaMemcpyAsync(dt.p, t_start.data(), 4 * G, cudaMemcpyHostToDevice, st));
  k_snap<<<grid_for(G, 128), 128, 0, st>>>(view(cv), G, dt.p, dpos.p, dh.p, dc.p);
  ctx->own_launches++;
  std::vector<int64_t> pos(G);
  std::vector<uint64_t> hg(G), cg(G);
  std::vector<Move> mv(G);
  KCUDA(ctx, cudaMemcpyAsync(pos.data(), dpos.p, 8 * G, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaMemcpyAsync(hg.data(), dh.p, 8 * G, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaMemcpyAsync(cg.data(), dc.p, 8 * G, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaStreamSynchronize(st));
  hits = 0;
  cost = 0;
  for (int g = 0; g < G; g++) { hits += hg[g]; cost += cg[g]; }
  for (int phase = 0; phase < 2; phase++) {  // 0: (b) restore feasibility, 1: (c) ascend
    const bool up = phase == 1;
    if (up && cost > B) break;
    for (;;) {
      if (!up && cost <= B) break;
      KCUDA(ctx, cudaMemcpyAsync(dpos.p, pos.data(), 8 * G, cudaMemcpyHostToDevice, st));
      KCUDA(ctx, cudaMemcpyAsync(dh.p, hg.data(), 8 * G, cudaMemcpyHostToDevice, st));
      KCUDA(ctx, cudaMemcpyAsync(dc.p, cg.data(), 8 * G, cudaMemcpyHostToDevice, st));
      k_best_move<<<G, 256, 0, st>>>(view(cv), G, up ? 1 : 0, dpos.p, dh.p, dc.p, up ? B - cost : 0, dmv.p);
      ctx->own_launches++;
      KCUDA(ctx, cudaMemcpyAsync(mv.data(), dmv.p, sizeof(Move) * G, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      int bg = -1;
      for (int g = 0; g < G; g++)
        if (host_better(up, mv[g], bg < 0 ? Move{0, 0, -2} : mv[bg])) bg = g;
      if (bg < 0) break;
      const Move &m = mv[bg];
      pos[bg] = m.row;
      if (up) { hg[bg] += m.dh; cg[bg] += m.dc; hits += m.dh; cost += m.dc; }
      else { hg[bg] -= m.dh; cg[bg] -= m.dc; hits -= m.dh; cost -= m.dc; }
    }
  }
  t_out.assign(G, 0);
  if (cost > B) {
    hits = 0;
    cost = 0;
    return KARETO_OK;
  }
  // the TTL of each row
  for (int g = 0; g < G; g++) {
    if (pos[g] >= cv.hfirst[g]) {
      KCUDA(ctx, cudaMemcpyAsync(&t_out[g], cv.v.p + pos[g], 4, cudaMemcpyDeviceToHost, st));
    }
  }
  return sync(ctx, "ttl local solve");
}

static uint64_t fmix64h(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

static kareto_status roi(kareto_ctx *ctx, const Curves &cv, std::vector<uint32_t> &t, std::vector<uint64_t> &h,
                         std::vector<uint64_t> &c) {
  const int G = cv.G;
  DBuf<uint32_t> dt;
  DBuf<uint64_t> dh, dc;
  KTRY(dt.alloc(ctx, G)); KTRY(dh.alloc(ctx, G)); KTRY(dc.alloc(ctx, G));
  {
    Pass ps(ctx, "F2_roi", 1, 1);
    k_roi<<<G, 256, 0, ctx->stream>>>(view(cv), G, dt.p, dh.p, dc.p);
  }
  t.resize(G); h.resize(G); c.resize(G);
  KCUDA(ctx, cudaMemcpyAsync(t.data(), dt.p, 4 * G, cudaMemcpyDeviceToHost, ctx->stream));
  KCUDA(ctx, cudaMemcpyAsync(h.data(), dh.p, 8 * G, cudaMemcpyDeviceToHost, ctx->stream));
  KCUDA(ctx, cudaMemcpyAsync(c.data(), dc.p, 8 * G, cudaMemcpyDeviceToHost, ctx->stream));
  return sync(ctx, "ttl roi");
}

}  // namespace kareto

using namespace kareto;

extern "C" kareto_status kareto_ttl_roi(kareto_ctx *ctx, const kareto_trace *tr, uint32_t *t_roi, uint64_t *h_roi,
                                        uint64_t *c_roi) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  if (tr && tr->sharded)
    return kareto::fail(ctx, KARETO_E_UNSUPPORTED, "%s needs the whole trace (not a time shard)", "kareto_ttl_roi");
  cudaSetDevice(ctx->device);
  if (!tr || !t_roi) return fail(ctx, KARETO_E_INVALID, "ttl_roi: null argument");
  Curves cv;
  KTRY(build_curves(ctx, tr, cv));
  std::vector<uint32_t> t;
  std::vector<uint64_t> h, c;
  KTRY(roi(ctx, cv, t, h, c));
  for (int g = 0; g < cv.G; g++) {
    t_roi[g] = t[g];
    if (h_roi) h_roi[g] = h[g];
    if (c_roi) c_roi[g] = c[g];
  }
  return KARETO_OK;
}

extern "C" kareto_status kareto_ttl_eval(kareto_ctx *ctx, const kareto_trace *tr, const uint32_t *ttl, int64_t n,
                                         uint64_t *hits, uint64_t *cost) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  if (tr && tr->sharded)
    return kareto::fail(ctx, KARETO_E_UNSUPPORTED, "%s needs the whole trace (not a time shard)", "kareto_ttl_eval");
  cudaSetDevice(ctx->device);
  if (!tr || n < 0 || (n > 0 && (!ttl || !hits || !cost))) return fail(ctx, KARETO_E_INVALID, "ttl_eval: bad arguments");
  const int G = tr->K + 1;
  for (int64_t i = 0; i < n * G; i++)
    if (ttl[i] == KARETO_TTL_INF) return fail(ctx, KARETO_E_INVALID, "ttl_eval: infinite TTL at [%lld][%lld]",
                                              (long long)(i / G), (long long)(i % G));
  if (n == 0) return KARETO_OK;
  Curves cv;
  KTRY(build_curves(ctx, tr, cv));
  cudaStream_t st = ctx->stream;
  DBuf<uint32_t> dt;
  DBuf<unsigned long long> dh, dc;
  KTRY(dt.alloc(ctx, n * G)); KTRY(dh.alloc(ctx, n)); KTRY(dc.alloc(ctx, n));
  KCUDA(ctx, cudaMemcpyAsync(dt.p, ttl, 4 * n * G, cudaMemcpyHostToDevice, st));
  KTRY(dh.zero()); KTRY(dc.zero());
  {
    Pass ps(ctx, "F2_eval", 1, 1);
    k_ttl_eval<<<grid_for(n * G, 256, 8 * ctx->num_sms), 256, 0, st>>>(view(cv), G, dt.p, n, dh.p, dc.p);
  }
  KCUDA(ctx, cudaMemcpyAsync(hits, dh.p, 8 * n, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaMemcpyAsync(cost, dc.p, 8 * n, cudaMemcpyDeviceToHost, st));
  return sync(ctx, "ttl eval");
}

extern "C" kareto_status kareto_ttl_allocate(kareto_ctx *ctx, const kareto_trace *tr, uint64_t budget, uint64_t seed,
                                             uint32_t *t_out, uint64_t *hits_out, uint64_t *cost_out,
                                             uint32_t *t_roi_out, uint32_t *t_init_out) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  if (tr && tr->sharded)
    return kareto::fail(ctx, KARETO_E_UNSUPPORTED, "%s needs the whole trace (not a time shard)", "kareto_ttl_allocate");
  cudaSetDevice(ctx->device);
  if (!tr || !t_out || !hits_out || !cost_out) return fail(ctx, KARETO_E_INVALID, "ttl_allocate: null argument");
  Curves cv;
  KTRY(build_curves(ctx, tr, cv));
  const int G = cv.G, K = G - 1;
  // l.2-7: per-group ROI-optimal TTL
  std::vector<uint32_t> t_roi;
  std::vector<uint64_t> h_roi, c_roi;
  KTRY(roi(ctx, cv, t_roi, h_roi, c_roi));
  // l.8-10: budget-aware scaling (R46)
  uint64_t c_un = 0;
  for (int g = 0; g < G; g++) c_un += c_roi[g];
  std::vector<uint32_t> t_init(G, 0);
  if (c_un > 0) {
    const double alpha = (double)budget / (double)c_un;
    for (int g = 0; g < G; g++) {
      const double x = std::floor(alpha * (double)t_roi[g]);
      t_init[g] = x >= (double)TTL_MAX_MS ? TTL_MAX_MS : (uint32_t)x;
    }
  }
  // l.11-13: starts (R45)
  std::vector<std::vector<uint32_t>> P{t_init};
  int sq = 0;
  while ((sq + 1) * (sq + 1) <= K) sq++;
  for (int s = 1; s <= sq; s++) {
    std::vector<uint32_t> row(G);
    for (int g = 0; g < G; g++) {
      const uint64_t u = fmix64h(seed * 1000003ull + 64ull * (uint64_t)s + (uint64_t)g);
      row[g] = (uint32_t)(((u128)t_init[g] * (((u128)1 << 63) + (u128)u)) >> 64);
    }
    P.push_back(row);
  }
  // R54: one more start, the largest uniform TTL within the budget (sum_g C_g(t) is
  // non-decreasing in t: binary search, one batched evaluation of 64 probes per round)
  {
    const int NP = 64;
    DBuf<uint32_t> dt;
    DBuf<unsigned long long> dh, dc;
    KTRY(dt.alloc(ctx, (int64_t)NP * G)); KTRY(dh.alloc(ctx, NP)); KTRY(dc.alloc(ctx, NP));
    std::vector<uint32_t> probe((size_t)NP * G);
    std::vector<unsigned long long> pc(NP);
    uint64_t lo = 0, hi = TTL_MAX_MS;  // invariant: C(lo) <= B (C(0) = 0), answer in [lo, hi]
    while (lo < hi) {
      // NP probes spread over (lo, hi]: the largest feasible one becomes lo, the next one - 1 hi
      uint64_t q[NP];
      for (int i = 0; i < NP; i++) q[i] = lo + ((hi - lo) * (uint64_t)(i + 1) + NP - 1) / NP;
      for (int i = 0; i < NP; i++)
        for (int g = 0; g < G; g++) probe[(size_t)i * G + g] = (uint32_t)q[i];
      KCUDA(ctx, cudaMemcpyAsync(dt.p, probe.data(), 4ull * NP * G, cudaMemcpyHostToDevice, ctx->stream));
      KTRY(dh.zero()); KTRY(dc.zero());
      k_ttl_eval<<<grid_for((int64_t)NP * G, 256), 256, 0, ctx->stream>>>(view(cv), G, dt.p, NP, dh.p, dc.p);
      ctx->own_launches++;
      KCUDA(ctx, cudaMemcpyAsync(pc.data(), dc.p, 8ull * NP, cudaMemcpyDeviceToHost, ctx->stream));
      KTRY(sync(ctx, "ttl uniform start"));
      uint64_t nlo = lo, nhi = hi;
      for (int i = 0; i < NP; i++) {
        if (pc[i] <= budget) nlo = q[i];
        else { nhi = q[i] - 1; break; }
      }
      lo = nlo; hi = nhi;
    }
    P.push_back(std::vector<uint32_t>(G, (uint32_t)lo));
  }
  // l.14-21: local solves, keep the most hits
  std::vector<uint32_t> best(G, 0), sol;
  uint64_t best_h = 0, best_c = 0;
  {
    Pass ps(ctx, "F2_local_solve", 0, 0);
    for (auto &ts : P) {
      uint64_t h = 0, c = 0;
      KTRY(local_solve(ctx, cv, ts, budget, sol, h, c));
      if (h > best_h) { best = sol; best_h = h; best_c = c; }
    }
  }
  for (int g = 0; g < G; g++) {
    t_out[g] = best[g];
    if (t_roi_out) t_roi_out[g] = t_roi[g];
    if (t_init_out) t_init_out[g] = t_init[g];
  }
  *hits_out = best_h;
  *cost_out = best_c;
  return KARETO_OK;
}

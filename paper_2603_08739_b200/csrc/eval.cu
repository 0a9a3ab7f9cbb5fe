// eval.cu -- kareto_eval_grid: rows a5 (K4 grid histograms), a6/a8 (K5+K7, objective.cu),
// multi-GPU sharding + NCCL allgather (row e).
//
// Stack path: for LRU configurations in TTL mode,
// or in CAPACITY mode with a uniform disk TTL, every count is a closed form of the
// per-access quantities (d, D = d + n-1-k, delta, group, k):
//   h1 = #{d <= c1}, h2 = #{c1 < d <= c12}, h3 = #{c12 < d <= C, delta <= tau}   (CAPACITY)
//   h3 = sum_g #{d > c12, delta <= tau_g, g}                                   (TTL mode)
//   e_t = #{D > b_t} - min(b_t, U);  writes / byte-time from the delta CDFs.
// K4 builds, in ONE pass over the accesses, histograms of d (and delta) over the sorted set
// of distinct boundaries used by the configurations of this rank's shard, privatised in
// shared memory; inclusive scans turn them into cumulative tables; K5+K7 evaluates every
// configuration from O(1) table lookups.
#include <algorithm>
#include <cub/cub.cuh>

#include "eval.cuh"
#include "replay.cuh"

namespace kareto {

constexpr int H_THREADS = 1024;
constexpr int LUT_BITS = 12;                 // boundary lookup table: 4096 buckets
constexpr int SMEM_BUDGET = 200 * 1024;
constexpr int SMEM_MAX = 227 * 1024;         // sm_100 max dynamic shared memory per block

// bucket LUT: lut[b] = first boundary index with Bd[i] >= (b << sh); lut[nbk] = nb
__global__ void k_build_lut(const uint32_t *__restrict__ Bd, int nb, int sh, uint32_t *__restrict__ lut) {
  int nbk = 1 << LUT_BITS;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= nbk; b += gridDim.x * blockDim.x) {
    uint64_t v = (uint64_t)b << sh;
    int lo = 0, hi = nb;
    while (lo < hi) {
      int m = (lo + hi) >> 1;
      if ((uint64_t)Bd[m] >= v) hi = m; else lo = m + 1;
    }
    lut[b] = (uint32_t)lo;
  }
}

// index of the first boundary >= v (nb if none)
__device__ __forceinline__ int bin_of(uint32_t v, const uint32_t *__restrict__ Bd, int nb, const uint32_t *lut_s,
                                      int sh) {
  uint32_t b = v >> sh;
  if (b >= (1u << LUT_BITS)) return nb;
  int lo = lut_s[b], hi = lut_s[b + 1];
  while (lo < hi) {
    int m = (lo + hi) >> 1;
    if (__ldg(&Bd[m]) >= v) hi = m; else lo = m + 1;
  }
  return lo;
}

__device__ __forceinline__ int tbin_of(uint32_t dl, const uint32_t *__restrict__ T, int nt) {
  int lo = 0, hi = nt;
  while (lo < hi) {
    int m = (lo + hi) >> 1;
    if (__ldg(&T[m]) >= dl) hi = m; else lo = m + 1;
  }
  return lo;
}

// K4a: histogram of (d-bin, tau-bin) with count and sum k, privatised in smem
// (cells [tc][bd] restricted to the window [c_lo, c_hi)), flushed with atomics.
// Per-access arrays are indexed by j - pos0 for positions j in [pos0, pos0 + N) (pos0 = 0 for a
// whole trace, the shard's first position for a time-sharded one).
__global__ void __launch_bounds__(H_THREADS) k_hist_d(uint64_t N, uint32_t pos0, uint64_t per_cta, const uint32_t *__restrict__ depth,
                                                      const uint32_t *__restrict__ req, const uint32_t *__restrict__ s,
                                                      const uint32_t *__restrict__ delta,
                                                      const uint32_t *__restrict__ Bd, int nb,
                                                      const uint32_t *__restrict__ lut, int sh,
                                                      const uint32_t *__restrict__ Tc, int ntc, int c_lo, int c_hi,
                                                      unsigned long long *__restrict__ gcnt,
                                                      unsigned long long *__restrict__ gsk) {
  extern __shared__ uint32_t sm[];
  uint32_t *lut_s = sm;                                  // (1<<LUT_BITS) + 1
  uint32_t *cnt = lut_s + (1 << LUT_BITS) + 1;
  const int W = c_hi - c_lo;
  uint32_t *sk = cnt + W;
  for (int i = threadIdx.x; i <= (1 << LUT_BITS); i += blockDim.x) lut_s[i] = lut[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) { cnt[i] = 0; sk[i] = 0; }
  __syncthreads();
  uint64_t j0 = blockIdx.x * per_cta, j1 = j0 + per_cta < N ? j0 + per_cta : N;
  for (uint64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    uint32_t d = depth[j];
    if (d == kNone) continue;
    int bd = bin_of(d, Bd, nb, lut_s, sh);
    if (bd >= nb) continue;
    int tc = ntc > 0 ? tbin_of(delta[j], Tc, ntc) : 0;
    int cell = tc * nb + bd - c_lo;
    if (cell < 0 || cell >= W) continue;
    uint32_t r = req[j];
    uint32_t k = s[r + 1] - 1 - ((uint32_t)j + pos0);
    atomicAdd(&cnt[cell], 1u);
    if (k) atomicAdd(&sk[cell], k);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    if (cnt[i]) atomicAdd(&gcnt[c_lo + i], (unsigned long long)cnt[i]);
    if (sk[i]) atomicAdd(&gsk[c_lo + i], (unsigned long long)sk[i]);
  }
}

// K4 fused (when both histograms fit in shared memory): one pass over the accesses builds
// the (d-bin, tau-bin) count / sum-k histogram and the D-bin count histogram (shared-memory
// atomics; warp aggregation by match_any measured slower here).
__global__ void __launch_bounds__(H_THREADS) k_hist_dD(uint64_t N, uint32_t pos0, uint64_t per_cta, const uint32_t *__restrict__ depth,
                                                       const uint32_t *__restrict__ req, const uint32_t *__restrict__ s,
                                                       const uint32_t *__restrict__ delta,
                                                       const uint32_t *__restrict__ Bd, int nb,
                                                       const uint32_t *__restrict__ lut, int sh,
                                                       const uint32_t *__restrict__ Tc, int ntc,
                                                       unsigned long long *__restrict__ gcnt,
                                                       unsigned long long *__restrict__ gsk,
                                                       unsigned long long *__restrict__ gD) {
  extern __shared__ uint32_t sm[];
  uint32_t *lut_s = sm;
  const int W = (ntc + 1) * nb;
  uint32_t *cnt = lut_s + (1 << LUT_BITS) + 1;
  uint32_t *sk = cnt + W;
  uint32_t *cD = sk + W;
  for (int i = threadIdx.x; i <= (1 << LUT_BITS); i += blockDim.x) lut_s[i] = lut[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) { cnt[i] = 0; sk[i] = 0; }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) cD[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  (void)lane;
  uint64_t j0 = blockIdx.x * per_cta, j1 = j0 + per_cta < N ? j0 + per_cta : N;
  // HD_U accesses per thread per round, loads issued breadth-first (depth/req, then the request
  // starts, then the boundary searches) so that a thread keeps several global loads in flight
  constexpr int HD_U = 4;
  for (uint64_t jb = j0; jb < j1; jb += (uint64_t)HD_U * blockDim.x) {
    uint32_t d[HD_U], r[HD_U], sr[HD_U], sr1[HD_U], dl[HD_U];
#pragma unroll
    for (int u = 0; u < HD_U; u++) {
      const uint64_t j = jb + (uint64_t)u * blockDim.x + threadIdx.x;
      d[u] = j < j1 ? depth[j] : kNone;
      r[u] = (d[u] != kNone) ? req[j] : 0u;
      dl[u] = (d[u] != kNone && ntc > 0) ? delta[j] : 0u;
    }
#pragma unroll
    for (int u = 0; u < HD_U; u++) {
      sr[u] = d[u] != kNone ? s[r[u]] : 0u;
      sr1[u] = d[u] != kNone ? s[r[u] + 1] : 0u;
    }
#pragma unroll
    for (int u = 0; u < HD_U; u++) {
      if (d[u] == kNone) continue;
      const uint32_t j = (uint32_t)(jb + (uint64_t)u * blockDim.x + threadIdx.x) + pos0;
      const uint32_t k = sr1[u] - 1 - j;
      const int bd = bin_of(d[u], Bd, nb, lut_s, sh);
      if (bd < nb) {
        const int cell = (ntc > 0 ? tbin_of(dl[u], Tc, ntc) : 0) * nb + bd;
        atomicAdd(&cnt[cell], 1u);
        if (k) atomicAdd(&sk[cell], k);
      }
      const uint32_t D = d[u] + (j - sr[u]);
      // D >= d: walk forward from d's bin (D - d is the offset inside the request, usually
      // small against the boundary gaps), falling back to the search after a few steps
      int bD = bd;
      int steps = 0;
      while (bD < nb && __ldg(&Bd[bD]) < D && steps < 4) { bD++; steps++; }
      if (bD < nb && __ldg(&Bd[bD]) < D) bD = bin_of(D, Bd, nb, lut_s, sh);
      if (bD < nb) atomicAdd(&cD[bD], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    if (cnt[i]) atomicAdd(&gcnt[i], (unsigned long long)cnt[i]);
    if (sk[i]) atomicAdd(&gsk[i], (unsigned long long)sk[i]);
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (cD[i]) atomicAdd(&gD[i], (unsigned long long)cD[i]);
}

// first run index q in [0, M) with runs[q].x >= pos (M if none), found by the whole CTA: each
// round probes blockDim.x evenly spaced runs and keeps the gap holding the answer (~3 rounds)
__device__ int64_t cta_run_lower_bound(const uint4 *__restrict__ runs, int64_t M, uint32_t pos) {
  int64_t lo = 0, hi = M;  // the answer lies in [lo, hi]
  while (hi > lo) {
    const int64_t step = (hi - lo + blockDim.x - 1) / blockDim.x;
    const int64_t q = lo + (int64_t)threadIdx.x * step;
    const int c = __syncthreads_count(q < hi && __ldg(&runs[q].x) < pos);  // a prefix of the probes
    if (c == 0) break;
    const int64_t nlo = lo + (int64_t)(c - 1) * step + 1, nhi = lo + (int64_t)c * step;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  return lo;
}

// K4 over runs (whole traces; same cells as k_hist_dD).  Inside a K3 run j0..j0+L-1 of request
// r the pre-request depth falls by one per access (d = d0 - t), D = d + (j - s_r) = d0 + j0 - s_r
// is constant, and so is delta (the run's previous accesses are consecutive positions with
// consecutive chain positions, hence one earlier request).  A run therefore adds the arithmetic
// range [d0 - L + 1, d0] to the (d-bin, tau-bin) cells -- per bin the count and the closed-form
// sum of k = s_{r+1} - 1 - j -- and L to one D bin: ~2.4 runs per request instead of ~100
// accesses.  CTA c takes the runs starting in positions [c per, (c+1) per), so its accesses
// (< per + max_blocks) bound the shared u32 sums exactly as in k_hist_dD.
__global__ void __launch_bounds__(H_THREADS) k_hist_runs(uint64_t N, uint64_t per_cta, int64_t M,
                                                         const uint4 *__restrict__ runs,
                                                         const uint32_t *__restrict__ s,
                                                         const uint32_t *__restrict__ delta,
                                                         const uint32_t *__restrict__ Bd, int nb,
                                                         const uint32_t *__restrict__ lut, int sh,
                                                         const uint32_t *__restrict__ Tc, int ntc,
                                                         unsigned long long *__restrict__ gcnt,
                                                         unsigned long long *__restrict__ gsk,
                                                         unsigned long long *__restrict__ gD) {
  extern __shared__ uint32_t sm[];
  uint32_t *lut_s = sm;
  const int W = (ntc + 1) * nb;
  uint32_t *cnt = lut_s + (1 << LUT_BITS) + 1;
  uint32_t *sk = cnt + W;
  uint32_t *cD = sk + W;
  for (int i = threadIdx.x; i <= (1 << LUT_BITS); i += blockDim.x) lut_s[i] = lut[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) { cnt[i] = 0; sk[i] = 0; }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) cD[i] = 0;
  const uint64_t p0 = blockIdx.x * per_cta, p1 = p0 + per_cta < N ? p0 + per_cta : N;
  const int64_t q0 = cta_run_lower_bound(runs, M, (uint32_t)p0);
  const int64_t q1 = p1 >= N ? M : cta_run_lower_bound(runs, M, (uint32_t)p1);
  __syncthreads();
  for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
    const uint4 rn = __ldg(&runs[q]);
    const uint32_t j0 = rn.x, L = rn.y, d0 = rn.z, r = rn.w;
    const uint32_t sr = __ldg(&s[r]), sr1 = __ldg(&s[r + 1]);
    const int tc = ntc > 0 ? tbin_of(__ldg(&delta[j0]), Tc, ntc) : 0;
    // k of the access at depth x: t = d0 - x, k = (sr1 - 1 - j0) - t
    const int64_t koff = (int64_t)(sr1 - 1 - j0) - (int64_t)d0;
    uint32_t lo = d0 - (L - 1);
    const uint32_t hi = d0;
    for (int b = bin_of(lo, Bd, nb, lut_s, sh); b < nb; b++) {
      const uint32_t bnd = __ldg(&Bd[b]);  // bin b holds depths in (Bd[b-1], Bd[b]]
      const uint32_t top = hi < bnd ? hi : bnd;
      const uint32_t c = top - lo + 1;
      const uint64_t ksum = (uint64_t)((koff + lo) + (koff + top)) * c / 2;
      const int cell = tc * nb + b;
      atomicAdd(&cnt[cell], c);
      if (ksum) atomicAdd(&sk[cell], (uint32_t)ksum);
      if (top == hi) break;
      lo = top + 1;
    }
    const int bD = bin_of(d0 + (j0 - sr), Bd, nb, lut_s, sh);
    if (bD < nb) atomicAdd(&cD[bD], L);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    if (cnt[i]) atomicAdd(&gcnt[i], (unsigned long long)cnt[i]);
    if (sk[i]) atomicAdd(&gsk[i], (unsigned long long)sk[i]);
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (cD[i]) atomicAdd(&gD[i], (unsigned long long)cD[i]);
}

// K4b: histogram of D over the boundaries (count), window [b_lo, b_hi)
__global__ void __launch_bounds__(H_THREADS) k_hist_D(uint64_t N, uint32_t pos0, uint64_t per_cta, const uint32_t *__restrict__ depth,
                                                      const uint32_t *__restrict__ req, const uint32_t *__restrict__ s,
                                                      const uint32_t *__restrict__ Bd, int nb,
                                                      const uint32_t *__restrict__ lut, int sh, int b_lo, int b_hi,
                                                      unsigned long long *__restrict__ gD) {
  extern __shared__ uint32_t sm[];
  uint32_t *lut_s = sm;
  uint32_t *cnt = lut_s + (1 << LUT_BITS) + 1;
  const int W = b_hi - b_lo;
  for (int i = threadIdx.x; i <= (1 << LUT_BITS); i += blockDim.x) lut_s[i] = lut[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint64_t j0 = blockIdx.x * per_cta, j1 = j0 + per_cta < N ? j0 + per_cta : N;
  for (uint64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    uint32_t d = depth[j];
    if (d == kNone) continue;
    uint32_t D = d + ((uint32_t)j + pos0 - s[req[j]]);
    int bd = bin_of(D, Bd, nb, lut_s, sh) - b_lo;
    if (bd < 0 || bd >= W) continue;
    atomicAdd(&cnt[bd], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < W; i += blockDim.x)
    if (cnt[i]) atomicAdd(&gD[b_lo + i], (unsigned long long)cnt[i]);
}

// K4c (TTL mode): C2 histogram [(i12bin)*G + g][t] in global memory (count, sum k) and
// per-group delta sums SDg[g][t] privatised in smem.
__global__ void __launch_bounds__(256) k_hist_ttl(uint64_t N, uint32_t pos0, const uint32_t *__restrict__ depth,
                                                  const uint32_t *__restrict__ req, const uint32_t *__restrict__ s,
                                                  const uint32_t *__restrict__ delta, const uint16_t *__restrict__ grp,
                                                  const uint32_t *__restrict__ B12, int nb12,
                                                  const uint32_t *__restrict__ Tt, int ntt, int G,
                                                  unsigned long long *__restrict__ C2, unsigned long long *__restrict__ S2,
                                                  unsigned long long *__restrict__ SDg) {
  extern __shared__ unsigned long long sd[];  // G * (ntt+1)
  const int nt1 = ntt + 1;
  for (int i = threadIdx.x; i < G * nt1; i += blockDim.x) sd[i] = 0;
  __syncthreads();
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t d = depth[j];
    if (d == kNone) continue;
    uint32_t r = req[j];
    uint32_t k = s[r + 1] - 1 - ((uint32_t)j + pos0);
    int g = grp[r];
    uint32_t dl = delta[j];
    int t = tbin_of(dl, Tt, ntt);
    int i = tbin_of(d, B12, nb12);  // first c12 boundary >= d (nb12: none)
    size_t cell = ((size_t)i * G + g) * nt1 + t;
    atomicAdd(&C2[cell], 1ull);
    if (k) atomicAdd(&S2[cell], (unsigned long long)k);
    atomicAdd(&sd[g * nt1 + t], (unsigned long long)dl);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * nt1; i += blockDim.x)
    if (sd[i]) atomicAdd(&SDg[i], sd[i]);
}

// column-wise prefix helpers ---------------------------------------------------
// C1: flat inclusive sums over [tc][bd] -> per-column prefix, then prefix over tc
__global__ void k_col_fix(const unsigned long long *__restrict__ flat, int ncol, int nb,
                          unsigned long long *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncol * nb; i += gridDim.x * blockDim.x) {
    int tc = i / nb;
    unsigned long long base = tc > 0 ? flat[(size_t)tc * nb - 1] : 0ull;
    out[i] = flat[i] - base;
  }
}
// K4 cumulative tables in one launch (one CTA per table): out[tc][b] = sum over tc' <= tc and
// b' <= b of h[tc'][b'] -- a block scan over b per column (8 consecutive bins per thread) plus the
// previous column's prefix (each thread adds the values it wrote itself for the same bins);
// table 2 (D) has one column.
constexpr int CUM_THREADS = 1024, CUM_ITEMS = 8;
__global__ void __launch_bounds__(CUM_THREADS) k_cumulate_tables(const unsigned long long *__restrict__ hC,
                                                                 const unsigned long long *__restrict__ hS,
                                                                 const unsigned long long *__restrict__ hD, int ncol,
                                                                 int nb, unsigned long long *__restrict__ C1,
                                                                 unsigned long long *__restrict__ S1,
                                                                 unsigned long long *__restrict__ CD) {
  typedef cub::BlockScan<unsigned long long, CUM_THREADS> Scan;
  __shared__ typename Scan::TempStorage ts;
  const unsigned long long *h = blockIdx.x == 0 ? hC : blockIdx.x == 1 ? hS : hD;
  unsigned long long *out = blockIdx.x == 0 ? C1 : blockIdx.x == 1 ? S1 : CD;
  const int nc = blockIdx.x == 2 ? 1 : ncol;
  constexpr int TILE = CUM_THREADS * CUM_ITEMS;
  for (int tc = 0; tc < nc; tc++) {
    unsigned long long carry = 0;
    for (int b0 = 0; b0 < nb; b0 += TILE) {
      const int bt = b0 + threadIdx.x * CUM_ITEMS;  // this thread's first bin
      unsigned long long v[CUM_ITEMS], sum = 0;
#pragma unroll
      for (int k = 0; k < CUM_ITEMS; k++) {
        v[k] = bt + k < nb ? h[(size_t)tc * nb + bt + k] : 0ull;
        sum += v[k];
      }
      unsigned long long excl, tot;
      Scan(ts).ExclusiveSum(sum, excl, tot);
      unsigned long long run = carry + excl;
#pragma unroll
      for (int k = 0; k < CUM_ITEMS; k++) {
        run += v[k];
        if (bt + k < nb) {
          const size_t i = (size_t)tc * nb + bt + k;
          out[i] = run + (tc > 0 ? out[i - nb] : 0ull);
        }
      }
      carry += tot;
      __syncthreads();  // ts is reused
    }
  }
}

__global__ void k_prefix_over_cols(unsigned long long *__restrict__ a, int ncol, int nb) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    unsigned long long acc = 0;
    for (int tc = 0; tc < ncol; tc++) { acc += a[(size_t)tc * nb + b]; a[(size_t)tc * nb + b] = acc; }
  }
}
// C2 [i][g][t]: prefix over i (per g,t), then over t (per i,g); SDg prefix over t
__global__ void k_prefix_c2_i(unsigned long long *__restrict__ a, int ni, int G, int nt1) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < G * nt1; x += gridDim.x * blockDim.x) {
    unsigned long long acc = 0;
    for (int i = 0; i < ni; i++) { acc += a[(size_t)i * G * nt1 + x]; a[(size_t)i * G * nt1 + x] = acc; }
  }
}
__global__ void k_prefix_t(unsigned long long *__restrict__ a, int rows, int nt1) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < rows; x += gridDim.x * blockDim.x) {
    unsigned long long acc = 0;
    for (int t = 0; t < nt1; t++) { acc += a[(size_t)x * nt1 + t]; a[(size_t)x * nt1 + t] = acc; }
  }
}

// boundary values of the stack configurations (clamped to U; C unused in TTL mode), and
// the c12 values of TTL-mode configurations (kNone sentinel for CAPACITY ones)
__device__ __forceinline__ uint64_t sat_add_d(uint64_t a, uint64_t b) { return a > ~0ull - b ? ~0ull : a + b; }
__global__ void k_bound_vals(const kareto_config *__restrict__ c, int64_t n, uint64_t U, uint32_t *__restrict__ vals,
                             uint32_t *__restrict__ v12) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const kareto_config x = c[i];
    uint64_t c12 = sat_add_d(x.cap[0], x.cap[1]);
    bool ttl = x.cap[2] == KARETO_INF;
    uint64_t C = ttl ? c12 : sat_add_d(c12, x.cap[2]);
    vals[3 * i] = (uint32_t)(x.cap[0] < U ? x.cap[0] : U);
    vals[3 * i + 1] = (uint32_t)(c12 < U ? c12 : U);
    vals[3 * i + 2] = (uint32_t)(C < U ? C : U);
    v12[i] = ttl ? (uint32_t)(c12 < U ? c12 : U) : kNone;
  }
}
__device__ __forceinline__ int32_t lb32(const uint32_t *__restrict__ v, int n, uint32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) { int m = (lo + hi) >> 1; if (v[m] >= x) hi = m; else lo = m + 1; }
  return lo;
}
__global__ void k_cfgdev(const kareto_config *__restrict__ c, int64_t n, uint64_t U, const uint32_t *__restrict__ Bd,
                         int nb, const uint32_t *__restrict__ B12, int nb12, const uint32_t *__restrict__ Tc, int ntc,
                         const uint32_t *__restrict__ rows, int n_tuner, int G, CfgDev *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const kareto_config x = c[i];
    auto cl = [&](uint64_t v) { return (uint32_t)(v < U ? v : U); };
    uint64_t c12 = sat_add_d(x.cap[0], x.cap[1]);
    int ri = n_tuner > 0 ? x.tuner : 0;
    CfgDev d{};
    d.i1 = lb32(Bd, nb, cl(x.cap[0]));
    d.i12 = lb32(Bd, nb, cl(c12));
    d.row = ri;
    if (x.cap[2] != KARETO_INF) {
      d.iC = lb32(Bd, nb, cl(sat_add_d(c12, x.cap[2])));
      uint32_t tau = rows[(size_t)ri * G];
      d.tc = tau == KARETO_TTL_INF ? ntc : lb32(Tc, ntc, tau);
      d.i12t = 0;
    } else {
      d.iC = -1;
      d.tc = ntc;
      d.i12t = lb32(B12, nb12, cl(c12));
    }
    out[i] = d;
  }
}

__global__ void k_scatter_out(const kareto_counts *__restrict__ c, const double *__restrict__ o,
                              const uint32_t *__restrict__ idx, int64_t n, kareto_counts *__restrict__ cout,
                              double *__restrict__ oout) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t d = idx[i];
    cout[d] = c[i];
    oout[3 * (size_t)d] = o[3 * i];
    oout[3 * (size_t)d + 1] = o[3 * i + 1];
    oout[3 * (size_t)d + 2] = o[3 * i + 2];
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

template <typename T>
static kareto_status upload(kareto_ctx *ctx, DBuf<T> &b, const std::vector<T> &v) {
  KTRY(b.alloc(ctx, v.size() ? v.size() : 1));
  if (!v.empty()) KCUDA(ctx, cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return KARETO_OK;
}

static bool model_valid(const kareto_model *m) {
  if (m->instances < 1 || m->gpus_per_instance < 1 || m->block_bytes < 1 || !(m->bw_dram > 0)) return false;
  if (m->n_media < 1 || m->n_media > 8 || m->n_phi < 0 || m->n_phi > 8) return false;
  for (int i = 0; i < m->n_media; i++)
    if (!(m->media[i].bw_max > 0) || m->media[i].bw_base < 0 || m->media[i].bw_slope < 0 || m->media[i].price < 0)
      return false;
  for (int i = 1; i < m->n_phi; i++)
    if (!(m->phi[i].breakpoint > m->phi[i - 1].breakpoint)) return false;
  if (m->n_phi > 0 && m->phi[0].breakpoint != 0.0) return false;
  if (m->c_hw < 0 || m->p_hbm < 0 || m->p_dram < 0 || m->iops_per_block < 0 || m->ttl_prov_gb < 0) return false;
  return true;
}

static inline uint64_t sat_add(uint64_t a, uint64_t b) { return a > UINT64_MAX - b ? UINT64_MAX : a + b; }

// deterministic contiguous shard of [0, n) for `rank` of `world`
static void shard_range(int64_t n, int rank, int world, int64_t &lo, int64_t &hi) {
  lo = n * rank / world;
  hi = n * (rank + 1) / world;
}

// Cost-weighted contiguous shards: a stack-path configuration costs O(1) on top of
// the trace passes every rank runs anyway (weight 1); a K6 replay configuration costs a pass over
// the trace, scaled by its class's relative pass time (replay.cu: list 1.0, FIFO/list + expiry
// wheel 2.2, LFU 1.95, LFU + expiry wheel 3.2, LRU + group expiry lists 2.27) -- weight 10^6 x that.
// bounds[r] = the largest i with world * prefix(i) <= r * total, so unit weights give exactly
// shard_range's floor(n r / world).  Every rank computes the same bounds from the same list.
static void shard_bounds(const kareto_config *cfg, int64_t n, const uint32_t *rows, int n_tuner, int G, int world,
                         int64_t *bounds) {
  const uint64_t stack_w = 1;
  const uint64_t class_w[5] = {1000000, 2200000, 1950000, 3200000, 2270000};
  std::vector<uint64_t> pre((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; i++) {
    const kareto_config &c = cfg[i];
    const uint32_t *tau = rows + (size_t)(n_tuner > 0 ? c.tuner : 0) * G;
    bool uniform = true, any_finite = false;
    for (int g = 0; g < G; g++) {
      uniform &= tau[g] == tau[0];
      any_finite |= tau[g] != KARETO_TTL_INF;
    }
    uint64_t w = stack_w;
    if (!(c.policy == KARETO_LRU && (c.cap[2] == KARETO_INF || uniform))) {
      const bool exp = c.cap[2] != KARETO_INF && any_finite;
      const int k = (exp && c.policy == KARETO_LRU) ? 4 : (c.policy == KARETO_LFU ? 2 : 0) + (exp ? 1 : 0);
      w = class_w[k];
    }
    pre[i + 1] = pre[i] + w;
  }
  const unsigned __int128 total = pre[n];
  bounds[0] = 0;
  int64_t i = 0;
  for (int r = 1; r < world; r++) {
    const unsigned __int128 target = total * (unsigned)r;
    while (i < n && (unsigned __int128)pre[i + 1] * (unsigned)world <= target) i++;
    bounds[r] = i;
  }
  bounds[world] = n;
}

#include <chrono>
#define HT(name)                                                                                          \
  do {                                                                                                    \
    if (ht_on) {                                                                                          \
      auto t_ = std::chrono::steady_clock::now();                                                         \
      fprintf(stderr, "[eval] %-10s %.3f ms\n", name, std::chrono::duration<double, std::milli>(t_ - ht0).count()); \
    }                                                                                                     \
  } while (0)
struct BoundCache {
  bool valid = false;
  uint64_t U = 0;
  int nb = 0, nb12 = 0;
  DBuf<uint32_t> dBd, dB12, dlut;
  DBuf<CfgDev> dcd;
};

// Everything kareto_eval_grid derives from the configuration list and the TTL table alone
// (validation, the shard, the stack / replay split, the TTL value sets, device copies): built once
// per call, or once per kareto_grid for repeated evaluation (kareto_grid_create).
struct GridPrep {
  int64_t n_cfg = 0;
  int G = 1, n_tuner = 0, nrows = 1;
  std::vector<uint32_t> rows;
  std::vector<char> row_uniform, row_finite;
  bool cfg_shard = false;
  std::vector<int64_t> bounds;
  int64_t lo = 0, hi = 0, ns = 0, nS = 0, nP = 0;
  std::vector<kareto_config> cP;   // replay configurations (host copy for K6)
  std::vector<uint32_t> iS, iP;    // their positions in the shard
  std::vector<uint32_t> Tc, Tt, tix;
  int ntc = 0, ntt = 0;
  // model-dependent checks, done per evaluation from these maxima
  int max_medium = -1;
  int64_t idx_medium = 0, idx_cap = 0;
  uint64_t max_capsum = 0;
  // device copies
  DBuf<kareto_config> dcfg, dcfgP;
  DBuf<uint32_t> dTc, dTt, dtix, drows, diS, diP;
  mutable BoundCache bc;  // K4 boundary sets for the last U evaluated
};

static kareto_status prep_grid(kareto_ctx *ctx, const kareto_config *cfg, int64_t n_cfg, const uint32_t *ttl_ms,
                               int32_t n_tuner, int G, bool cfg_shard, GridPrep &P) {
  cudaStream_t st = ctx->stream;
  if (n_cfg < 0 || (n_cfg > 0 && !cfg)) return fail(ctx, KARETO_E_INVALID, "bad arguments");
  if (n_tuner < 0 || (n_tuner > 0 && !ttl_ms)) return fail(ctx, KARETO_E_INVALID, "bad TTL table");
  P.n_cfg = n_cfg;
  P.G = G;
  P.n_tuner = n_tuner;
  P.cfg_shard = cfg_shard;
  // rows (an all-infinite row when no table is given)
  std::vector<uint32_t> &rows = P.rows;
  int &nrows = P.nrows;
  nrows = n_tuner;
  if (n_tuner == 0) { rows.assign(G, KARETO_TTL_INF); nrows = 1; }
  else rows.assign(ttl_ms, ttl_ms + (size_t)n_tuner * G);
  // per-row flags: uniform across groups, all finite
  std::vector<char> &row_uniform = P.row_uniform, &row_finite = P.row_finite;
  row_uniform.assign(nrows, 1);
  row_finite.assign(nrows, 1);
  for (int r = 0; r < nrows; r++)
    for (int g = 0; g < G; g++) {
      if (rows[(size_t)r * G + g] != rows[(size_t)r * G]) row_uniform[r] = 0;
      if (rows[(size_t)r * G + g] == KARETO_TTL_INF) row_finite[r] = 0;
    }
  // ---- validation (every rank validates the full list identically), O(1) per configuration
  for (int64_t i = 0; i < n_cfg; i++) {
    const kareto_config &c = cfg[i];
    if (c.policy > KARETO_LFU) return fail(ctx, KARETO_E_INVALID, "config %lld: policy %d", (long long)i, c.policy);
    if (n_tuner > 0 && c.tuner >= n_tuner) return fail(ctx, KARETO_E_INVALID, "config %lld: tuner", (long long)i);
    if (c.cap[0] == KARETO_INF || c.cap[1] == KARETO_INF)
      return fail(ctx, KARETO_E_INVALID, "config %lld: infinite HBM/DRAM", (long long)i);
    const int ri = n_tuner > 0 ? c.tuner : 0;
    const bool ttl = c.cap[2] == KARETO_INF;
    if (ttl && !row_finite[ri])
      return fail(ctx, KARETO_E_INVALID, "config %lld: TTL mode needs finite TTLs (R22)", (long long)i);
    if ((int)c.medium > P.max_medium) { P.max_medium = c.medium; P.idx_medium = i; }
    const uint64_t cs = ttl ? sat_add(c.cap[0], c.cap[1]) : sat_add(sat_add(c.cap[0], c.cap[1]), c.cap[2]);
    if (cs > P.max_capsum) { P.max_capsum = cs; P.idx_cap = i; }
  }
  // ---- shard
  int64_t &lo = P.lo, &hi = P.hi;
  lo = 0;
  hi = n_cfg;
  P.bounds.assign((size_t)ctx->world + 1, 0);
  if (cfg_shard) {
    shard_bounds(cfg, n_cfg, rows.data(), n_tuner, G, ctx->world, P.bounds.data());
    lo = P.bounds[ctx->rank];
    hi = P.bounds[ctx->rank + 1];
  }
  const int64_t ns = P.ns = hi - lo;
  const kareto_config *sc = cfg + lo;
  // stack-eligible (LRU, and TTL mode or a uniform disk TTL) vs per-configuration replay (K6)
  // (one counting pass; the split copies are only made when both kinds are present, otherwise
  // the caller's array is uploaded as it is)
  std::vector<kareto_config> cS;
  std::vector<char> cap_row_used(nrows, 0), ttl_row_used(nrows, 0);
  auto stack_ok = [&](const kareto_config &c) {
    const int ri = n_tuner > 0 ? c.tuner : 0;
    return c.policy == KARETO_LRU && (c.cap[2] == KARETO_INF || row_uniform[ri]);
  };
  int64_t nP = 0;
  for (int64_t i = 0; i < ns; i++) {
    const kareto_config &c = sc[i];
    const int ri = n_tuner > 0 ? c.tuner : 0;
    if (stack_ok(c)) (c.cap[2] == KARETO_INF ? ttl_row_used : cap_row_used)[ri] = 1;
    else nP++;
  }
  P.nP = nP;
  const int64_t nS = P.nS = ns - nP;
  const kareto_config *cSp = sc;  // the stack configurations, in shard order when nP == 0
  if (nP > 0) {
    cS.reserve(nS); P.iS.reserve(nS); P.cP.reserve(nP); P.iP.reserve(nP);
    for (int64_t i = 0; i < ns; i++) {
      if (stack_ok(sc[i])) { cS.push_back(sc[i]); P.iS.push_back((uint32_t)i); }
      else { P.cP.push_back(sc[i]); P.iP.push_back((uint32_t)i); }
    }
    cSp = cS.data();
  }
  // TTL value sets: uniform CAPACITY TTLs (Tc) and all TTLs of rows used in TTL mode (Tt)
  std::vector<uint32_t> &Tc = P.Tc, &Tt = P.Tt;
  for (int r = 0; r < nrows; r++) {
    if (cap_row_used[r] && rows[(size_t)r * G] != KARETO_TTL_INF) Tc.push_back(rows[(size_t)r * G]);
    if (ttl_row_used[r])
      for (int g = 0; g < G; g++) Tt.push_back(rows[(size_t)r * G + g]);
  }
  auto uniq = [](std::vector<uint32_t> &v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  };
  uniq(Tc); uniq(Tt);
  P.ntc = (int)Tc.size();
  P.ntt = (int)Tt.size();
  P.tix.assign((size_t)nrows * G, 0);
  for (int r = 0; r < nrows; r++)
    if (ttl_row_used[r])
      for (int g = 0; g < G; g++)
        P.tix[(size_t)r * G + g] =
            (uint32_t)(std::lower_bound(Tt.begin(), Tt.end(), rows[(size_t)r * G + g]) - Tt.begin());
  // device copies
  KTRY(upload(ctx, P.dTc, Tc)); KTRY(upload(ctx, P.dTt, Tt)); KTRY(upload(ctx, P.dtix, P.tix));
  KTRY(upload(ctx, P.drows, rows));
  KTRY(P.dcfg.alloc(ctx, nS > 0 ? nS : 1));
  if (nS > 0) KCUDA(ctx, cudaMemcpyAsync(P.dcfg.p, cSp, sizeof(kareto_config) * nS, cudaMemcpyHostToDevice, st));
  if (nP > 0) {
    KTRY(P.dcfgP.alloc(ctx, nP));
    KCUDA(ctx, cudaMemcpyAsync(P.dcfgP.p, P.cP.data(), sizeof(kareto_config) * nP, cudaMemcpyHostToDevice, st));
    KTRY(upload(ctx, P.diS, P.iS)); KTRY(upload(ctx, P.diP, P.iP));
  }
  return KARETO_OK;
}

static kareto_status run_eval(kareto_ctx *ctx, const kareto_trace *tr, const GridPrep &prep, const kareto_model *model,
                              kareto_counts *counts_out, double *obj_out, int32_t on_dev) {
  const bool ht_on = getenv("KARETO_HOST_TIMING") != nullptr;
  const auto ht0 = std::chrono::steady_clock::now();
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  if (!model) return fail(ctx, KARETO_E_INVALID, "bad arguments");
  if (!model_valid(model)) return fail(ctx, KARETO_E_INVALID, "invalid model constants");
  const int G = tr->K + 1;
  if (prep.G != G) return fail(ctx, KARETO_E_INVALID, "grid built for %d groups, trace has %d", prep.G, G);
  const uint64_t N = (uint64_t)tr->N, U = (uint64_t)tr->U;
  // a time-sharded trace (row f4) holds the accesses [pos_lo, pos_hi): every rank evaluates the
  // whole grid from histograms summed over the ranks (no configuration sharding, no gather)
  const bool tsh = tr->sharded;
  const uint64_t Nl = (uint64_t)(tr->pos_hi - tr->pos_lo);
  const uint32_t jb = (uint32_t)tr->pos_lo;
  const bool cfg_shard = prep.cfg_shard;
  const int64_t n_cfg = prep.n_cfg;
  const int n_tuner = prep.n_tuner;
  const std::vector<uint32_t> &rows = prep.rows;
  HT("start");
  // model-dependent checks from the grid's maxima (the per-configuration ones ran in prep_grid)
  if (n_cfg > 0 && prep.max_medium >= model->n_media)
    return fail(ctx, KARETO_E_INVALID, "config %lld: medium", (long long)prep.idx_medium);
  if (n_cfg > 0 && (unsigned __int128)prep.max_capsum * model->block_bytes > (unsigned __int128)UINT64_MAX)
    return fail(ctx, KARETO_E_OVERFLOW, "config %lld: capacity x block bytes", (long long)prep.idx_cap);
  // trace x model integer constants
  unsigned __int128 P0 = (unsigned __int128)model->alpha_ps * tr->SL + (unsigned __int128)model->beta_ps * tr->SQ;
  if (P0 > (unsigned __int128)UINT64_MAX) return fail(ctx, KARETO_E_OVERFLOW, "no-cache prefill cost >= 2^64 ps");
  if ((unsigned __int128)model->dec_ps * tr->O > (unsigned __int128)UINT64_MAX)
    return fail(ctx, KARETO_E_OVERFLOW, "decode cost >= 2^64 ps");
  if ((unsigned __int128)(2 * N + 2 * U) * model->block_bytes > (unsigned __int128)UINT64_MAX)
    return fail(ctx, KARETO_E_OVERFLOW, "transfer bytes >= 2^64");
  ModelConsts mc{(uint64_t)P0, (uint64_t)tr->R, N, U, tr->Ltok, tr->O, tr->span_ms};
  HT("validated");
  const std::vector<int64_t> &bounds = prep.bounds;
  const int64_t ns = prep.ns, nS = prep.nS, nP = prep.nP;
  const std::vector<kareto_config> &cP = prep.cP;
  if (tsh && nP > 0)
    return fail(ctx, KARETO_E_UNSUPPORTED,
                "time-sharded trace: %lld configurations need the per-configuration replay (FIFO, LFU, per-group "
                "TTL on a finite disk); load the whole trace for those", (long long)nP);
  const int ntc = prep.ntc, ntt = prep.ntt;
  const DBuf<uint32_t> &dTc = prep.dTc, &dTt = prep.dTt, &dtix = prep.dtix, &drows = prep.drows;
  const DBuf<kareto_config> &dcfg = prep.dcfg;

  HT("classified");
  // ---- boundary sets, their LUT and per-configuration lookup indices, on the GPU.  They depend
  // only on the grid and U (capacities are clamped to U), so a prepared grid keeps them for the
  // next evaluation against a trace with the same U (the planner's grid over trace after trace)
  DBuf<uint8_t> tmp;
  int sh = 0;
  while (((uint64_t)U >> sh) >= (1ull << LUT_BITS)) sh++;
  BoundCache &bc = prep.bc;
  if (!bc.valid || bc.U != U) {
    bc.valid = false;
    bc.nb = bc.nb12 = 0;
    KTRY(bc.dcd.alloc(ctx, nS > 0 ? nS : 1));
    KTRY(bc.dlut.alloc(ctx, (1 << LUT_BITS) + 1));
    if (nS > 0) {
      DBuf<uint32_t> vals, vals_s, v12, v12_s;
      DBuf<int> cnt;
      KTRY(vals.alloc(ctx, 3 * nS)); KTRY(vals_s.alloc(ctx, 3 * nS)); KTRY(v12.alloc(ctx, nS)); KTRY(v12_s.alloc(ctx, nS));
      KTRY(bc.dBd.alloc(ctx, 3 * nS)); KTRY(bc.dB12.alloc(ctx, nS)); KTRY(cnt.alloc(ctx, 2));
      Pass ps(ctx, "K4_boundaries", 1, 3);
      k_bound_vals<<<grid_for(nS, 256, 4 * sms), 256, 0, st>>>(dcfg.p, nS, U, vals.p, v12.p);
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortKeys(t, b, vals.p, vals_s.p, (int)(3 * nS), 0, 32, st);
      }));
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceSelect::Unique(t, b, vals_s.p, bc.dBd.p, cnt.p, (int)(3 * nS), st);
      }));
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortKeys(t, b, v12.p, v12_s.p, (int)nS, 0, 32, st);
      }));
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceSelect::Unique(t, b, v12_s.p, bc.dB12.p, cnt.p + 1, (int)nS, st);
      }));
      int hc[2] = {0, 0};
      uint32_t last12 = 0;
      KCUDA(ctx, cudaMemcpyAsync(hc, cnt.p, 8, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      bc.nb = hc[0];
      bc.nb12 = hc[1];
      if (bc.nb12 > 0) {  // drop the sentinel of CAPACITY configurations (the largest key)
        KCUDA(ctx, cudaMemcpyAsync(&last12, bc.dB12.p + bc.nb12 - 1, 4, cudaMemcpyDeviceToHost, st));
        KCUDA(ctx, cudaStreamSynchronize(st));
        if (last12 == kNone) bc.nb12--;
      }
      k_cfgdev<<<grid_for(nS, 256, 4 * sms), 256, 0, st>>>(dcfg.p, nS, U, bc.dBd.p, bc.nb, bc.dB12.p, bc.nb12, dTc.p,
                                                           ntc, drows.p, n_tuner, G, bc.dcd.p);
      if (bc.nb > 0) k_build_lut<<<grid_for((1 << LUT_BITS) + 1, 256), 256, 0, st>>>(bc.dBd.p, bc.nb, sh, bc.dlut.p);
    }
    bc.U = U;
    bc.valid = true;
  }
  const int nb = bc.nb, nb12 = bc.nb12;
  const DBuf<uint32_t> &dBd = bc.dBd, &dB12 = bc.dB12, &dlut = bc.dlut;
  const DBuf<CfgDev> &dcd = bc.dcd;

  HT("boundaries");
  // ---- K4: histograms over the accesses
  const int ncol = ntc + 1;
  DBuf<unsigned long long> hC, hS, hD, C1, S1, CD;
  size_t ncell = (size_t)ncol * (nb > 0 ? nb : 1);
  KTRY(hC.alloc(ctx, ncell)); KTRY(hS.alloc(ctx, ncell)); KTRY(hD.alloc(ctx, nb > 0 ? nb : 1));
  KTRY(hC.zero()); KTRY(hS.zero()); KTRY(hD.zero());
  KTRY(C1.alloc(ctx, ncell)); KTRY(S1.alloc(ctx, ncell)); KTRY(CD.alloc(ctx, nb > 0 ? nb : 1));
  KTRY(C1.zero()); KTRY(S1.zero()); KTRY(CD.zero());
  const uint32_t *depth = tr->depth, *req = tr->req, *s = tr->s, *delta = tr->delta;
  if (ns > 0 && N > 0 && nb > 0) {
    const uint64_t N = Nl;  // this rank's accesses
    // CTA ranges bounded so that per-CTA u32 sums of k cannot overflow
    uint64_t maxk = tr->max_blocks > 1 ? (uint64_t)tr->max_blocks - 1 : 1;
    uint64_t cap_per = 0xFFFFFFFFull / maxk;
    uint64_t per = (N + 2 * sms - 1) / (2 * sms);
    if (per > cap_per) per = cap_per;
    if (per < 1) per = 1;
    unsigned g = (unsigned)((N + per - 1) / per);
    const size_t lut_bytes = 4 * ((1 << LUT_BITS) + 1);
    const int wcell = (int)((SMEM_BUDGET - lut_bytes) / 8);
    const int wD = (int)((SMEM_BUDGET - lut_bytes) / 4);
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(k_hist_d, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET);
      cudaFuncSetAttribute(k_hist_D, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET);
      cudaFuncSetAttribute(k_hist_dD, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
      attr_set = true;
    }
    const size_t fused = lut_bytes + 8 * ncell + 4 * (size_t)nb;
    // whole traces: one pass over the K3 runs (d falls by one per access inside a run)
    const uint64_t maxb = tr->max_blocks > 0 ? (uint64_t)tr->max_blocks : 1;
    const bool by_runs = !tsh && tr->runs && tr->n_runs > 0 && cap_per > maxb + 1 &&
                         getenv("KARETO_K4_ACCESS") == nullptr;
    if (fused <= (size_t)SMEM_MAX && by_runs) {
      static bool attr_runs = false;
      if (!attr_runs) {
        cudaFuncSetAttribute(k_hist_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
        attr_runs = true;
      }
      uint64_t per_r = (N + sms - 1) / sms;  // one CTA per SM: half the cell flushes of k_hist_dD
      if (per_r > cap_per - maxb) per_r = cap_per - maxb;
      const unsigned gr = (unsigned)((N + per_r - 1) / per_r);
      Pass ps(ctx, "K4_hist_runs", 1, 1);
      k_hist_runs<<<gr, H_THREADS, fused, st>>>(N, per_r, tr->n_runs, tr->runs, s, delta, dBd.p, nb, dlut.p, sh,
                                                dTc.p, ntc, hC.p, hS.p, hD.p);
    } else if (fused <= (size_t)SMEM_MAX) {  // one pass for both histograms
      KTRY(ensure_depth(ctx, const_cast<kareto_trace *>(tr)));
      Pass ps(ctx, "K4_hist_dD", 1, 1);
      if (N > 0) k_hist_dD<<<g, H_THREADS, fused, st>>>(N, jb, per, depth, req, s, delta, dBd.p, nb, dlut.p, sh, dTc.p, ntc, hC.p,
                                            hS.p, hD.p);
    } else {
    KTRY(ensure_depth(ctx, const_cast<kareto_trace *>(tr)));
    for (int c0 = 0; c0 < (int)ncell; c0 += wcell) {
      int c1 = c0 + wcell < (int)ncell ? c0 + wcell : (int)ncell;
      size_t smem = lut_bytes + 8 * (size_t)(c1 - c0);
      Pass ps(ctx, "K4_hist_d", 1, 1);
      if (N > 0) k_hist_d<<<g, H_THREADS, smem, st>>>(N, jb, per, depth, req, s, delta, dBd.p, nb, dlut.p, sh, dTc.p, ntc, c0, c1,
                                           hC.p, hS.p);
    }
    for (int b0 = 0; b0 < nb; b0 += wD) {
      int b1 = b0 + wD < nb ? b0 + wD : nb;
      size_t smem = lut_bytes + 4 * (size_t)(b1 - b0);
      Pass ps(ctx, "K4_hist_D", 1, 1);
      if (N > 0) k_hist_D<<<g, H_THREADS, smem, st>>>(N, jb, per, depth, req, s, dBd.p, nb, dlut.p, sh, b0, b1, hD.p);
    }
    }
    if (tsh) {  // sum the shards' histograms (one allreduce over NVLink)
      Pass ps(ctx, "F4_allreduce", 0, 3);
      KTRY(coll_allreduce_u64(ctx, hC.p, ncell));
      KTRY(coll_allreduce_u64(ctx, hS.p, ncell));
      KTRY(coll_allreduce_u64(ctx, hD.p, (size_t)nb));
    }
    {
      if (ncell <= (size_t)8 * CUM_THREADS * CUM_ITEMS) {  // small tables: one CTA per table
        Pass ps(ctx, "K4_cumulate", 1, 1);
        k_cumulate_tables<<<3, CUM_THREADS, 0, st>>>(hC.p, hS.p, hD.p, ncol, nb, C1.p, S1.p, CD.p);
      } else {
        Pass ps(ctx, "K4_cumulate", 0, 3);
        DBuf<unsigned long long> flat;
        KTRY(flat.alloc(ctx, ncell));
        KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
          return cub::DeviceScan::InclusiveSum(t, b, hC.p, flat.p, (int64_t)ncell, st);
        }));
        k_col_fix<<<grid_for(ncell, 256, 4 * sms), 256, 0, st>>>(flat.p, ncol, nb, C1.p);
        KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
          return cub::DeviceScan::InclusiveSum(t, b, hS.p, flat.p, (int64_t)ncell, st);
        }));
        k_col_fix<<<grid_for(ncell, 256, 4 * sms), 256, 0, st>>>(flat.p, ncol, nb, S1.p);
        k_prefix_over_cols<<<grid_for(nb, 256, 4 * sms), 256, 0, st>>>(C1.p, ncol, nb);
        k_prefix_over_cols<<<grid_for(nb, 256, 4 * sms), 256, 0, st>>>(S1.p, ncol, nb);
        KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
          return cub::DeviceScan::InclusiveSum(t, b, hD.p, CD.p, nb, st);
        }));
        ctx->own_launches += 4;
      }
    }
  }
  // TTL-mode tables
  const int nt1 = ntt + 1;
  DBuf<unsigned long long> C2, S2, SDg, dUg, dRg;
  size_t n2 = (size_t)(nb12 + 1) * G * nt1;
  KTRY(C2.alloc(ctx, n2)); KTRY(S2.alloc(ctx, n2)); KTRY(SDg.alloc(ctx, (size_t)G * nt1));
  KTRY(C2.zero()); KTRY(S2.zero()); KTRY(SDg.zero());
  std::vector<unsigned long long> hUg(G), hRg(G);
  for (int g = 0; g < G; g++) { hUg[g] = (unsigned long long)tr->U_g[g]; hRg[g] = (unsigned long long)tr->reuse_g[g]; }
  KTRY(upload(ctx, dUg, hUg)); KTRY(upload(ctx, dRg, hRg));
  if (ns > 0 && N > 0 && nb12 > 0) {
    KTRY(ensure_depth(ctx, const_cast<kareto_trace *>(tr)));
    size_t smem = 8 * (size_t)G * nt1;
    if (smem > 200 * 1024) return fail(ctx, KARETO_E_UNSUPPORTED, "too many groups x TTL values (%d x %d)", G, nt1);
    cudaFuncSetAttribute(k_hist_ttl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    {
      Pass ps(ctx, "K4_hist_ttl", 1, 1);
      if (Nl > 0)
        k_hist_ttl<<<grid_for(Nl, 256, 4 * sms), 256, smem, st>>>(Nl, jb, depth, req, s, delta, tr->grp, dB12.p, nb12,
                                                                  dTt.p, ntt, G, C2.p, S2.p, SDg.p);
    }
    if (tsh) {
      Pass ps(ctx, "F4_allreduce", 0, 3);
      KTRY(coll_allreduce_u64(ctx, C2.p, n2));
      KTRY(coll_allreduce_u64(ctx, S2.p, n2));
      KTRY(coll_allreduce_u64(ctx, SDg.p, (size_t)G * nt1));
    }
    Pass ps(ctx, "K4_cumulate_ttl", 1, 5);
    k_prefix_c2_i<<<grid_for(G * nt1, 256), 256, 0, st>>>(C2.p, nb12 + 1, G, nt1);
    k_prefix_c2_i<<<grid_for(G * nt1, 256), 256, 0, st>>>(S2.p, nb12 + 1, G, nt1);
    k_prefix_t<<<grid_for((nb12 + 1) * G, 256), 256, 0, st>>>(C2.p, (nb12 + 1) * G, nt1);
    k_prefix_t<<<grid_for((nb12 + 1) * G, 256), 256, 0, st>>>(S2.p, (nb12 + 1) * G, nt1);
    k_prefix_t<<<grid_for(G, 256), 256, 0, st>>>(SDg.p, G, nt1);
  }

  HT("k4");
  // ---- K5 + K7 on the shard
  DBuf<kareto_counts> dcounts;
  DBuf<double> dobj;
  int64_t nsa = ns > 0 ? ns : 1;
  // gathered outputs are assembled in padded per-rank slots: slot = the largest shard
  int64_t slot = nsa;
  if (cfg_shard) {
    slot = 1;
    for (int r = 0; r < ctx->world; r++) slot = std::max<int64_t>(slot, bounds[r + 1] - bounds[r]);
  }
  KTRY(dcounts.alloc(ctx, slot > 0 ? slot : 1)); KTRY(dobj.alloc(ctx, 3 * (slot > 0 ? slot : 1)));
  StackTables T{};
  T.Bd = nullptr; T.nb = nb; T.Tc = dTc.p; T.ntc = ntc;
  T.C1 = C1.p; T.S1 = S1.p; T.CD = CD.p;
  T.B12 = nullptr; T.nb12 = nb12; T.Tt = dTt.p; T.ntt = ntt; T.G = G;
  T.C2 = C2.p; T.S2 = S2.p; T.SDg = SDg.p; T.Ug = dUg.p; T.Rg = dRg.p;
  if (nP == 0) {  // pure stack shard: outputs in shard order directly
    launch_objective(ctx, T, dcfg.p, dcd.p, dtix.p, drows.p, nS, model, mc, nullptr, dcounts.p, dobj.p);
  } else {
    // K6 replay for the rest, then the objective from its counts; scatter both to shard order
    DBuf<kareto_counts> cntS, cntP;
    DBuf<double> objS, objP;
    KTRY(cntS.alloc(ctx, nS > 0 ? nS : 1)); KTRY(objS.alloc(ctx, 3 * (nS > 0 ? nS : 1)));
    KTRY(cntP.alloc(ctx, nP)); KTRY(objP.alloc(ctx, 3 * nP));
    launch_objective(ctx, T, dcfg.p, dcd.p, dtix.p, drows.p, nS, model, mc, nullptr, cntS.p, objS.p);
    KTRY(replay_eval(ctx, const_cast<kareto_trace *>(tr), cP.data(), nP, rows.data(), drows.p, n_tuner, cntP.p));
    launch_objective(ctx, T, prep.dcfgP.p, nullptr, dtix.p, drows.p, nP, model, mc, cntP.p, nullptr, objP.p);
    Pass ps(ctx, "K5_scatter", 1, 2);
    if (nS > 0) k_scatter_out<<<grid_for(nS, 256), 256, 0, st>>>(cntS.p, objS.p, prep.diS.p, nS, dcounts.p, dobj.p);
    k_scatter_out<<<grid_for(nP, 256), 256, 0, st>>>(cntP.p, objP.p, prep.diP.p, nP, dcounts.p, dobj.p);
  }

  HT("k57");
  // ---- gather (row e): one NCCL allgather of counts and objective vectors over NVLink
  kareto_counts *all_counts = dcounts.p;
  double *all_obj = dobj.p;
  DBuf<kareto_counts> gcounts;
  DBuf<double> gobj;
  if (cfg_shard) {
    const int W = ctx->world;
    KTRY(gcounts.alloc(ctx, (size_t)slot * W)); KTRY(gobj.alloc(ctx, (size_t)3 * slot * W));
    Pass ps(ctx, "K9_allgather", 0, 2);
    KTRY(coll_allgather(ctx, dcounts.p, gcounts.p, sizeof(kareto_counts) * slot));
    KTRY(coll_allgather(ctx, dobj.p, gobj.p, 24 * (size_t)slot));
    // compact rank slots into [0, n): rank r's shard occupies [lo_r, hi_r)
    DBuf<kareto_counts> ccounts;
    DBuf<double> cobj;
    KTRY(ccounts.alloc(ctx, n_cfg)); KTRY(cobj.alloc(ctx, 3 * n_cfg));
    for (int r = 0; r < W; r++) {
      const int64_t l = bounds[r], h = bounds[r + 1];
      if (h > l) {
        KCUDA(ctx, cudaMemcpyAsync(ccounts.p + l, gcounts.p + (size_t)r * slot, sizeof(kareto_counts) * (h - l),
                                   cudaMemcpyDeviceToDevice, st));
        KCUDA(ctx, cudaMemcpyAsync(cobj.p + 3 * l, gobj.p + (size_t)3 * r * slot, 24 * (h - l),
                                   cudaMemcpyDeviceToDevice, st));
      }
    }
    gcounts = std::move(ccounts);
    gobj = std::move(cobj);
    all_counts = gcounts.p;
    all_obj = gobj.p;
  }
  cudaMemcpyKind kind = on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (n_cfg > 0) {
    if (counts_out) KCUDA(ctx, cudaMemcpyAsync(counts_out, all_counts, sizeof(kareto_counts) * n_cfg, kind, st));
    if (obj_out) KCUDA(ctx, cudaMemcpyAsync(obj_out, all_obj, 24 * n_cfg, kind, st));
  }
  HT("copies");
  kareto_status sst = sync(ctx, "eval_grid");
  HT("synced");
  return sst;
}

static kareto_status eval(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg, int64_t n_cfg,
                          const uint32_t *ttl_ms, int32_t n_tuner, const kareto_model *model,
                          kareto_counts *counts_out, double *obj_out, int32_t on_dev) {
  if (!model) return fail(ctx, KARETO_E_INVALID, "bad arguments");
  GridPrep prep;
  const bool cfg_shard = (ctx->world > 1 || ctx->nccl) && !tr->sharded;
  KTRY(prep_grid(ctx, cfg, n_cfg, ttl_ms, n_tuner, tr->K + 1, cfg_shard, prep));
  return run_eval(ctx, tr, prep, model, counts_out, obj_out, on_dev);
}

kareto_status pareto_line_widths(kareto_ctx *ctx, const kareto_config *cfg, int64_t n, int *w, std::string *err);

}  // namespace kareto

extern "C" kareto_status kareto_grid_create(kareto_ctx *ctx, const kareto_config *cfg, int64_t n_cfg,
                                            const uint32_t *ttl_ms, int32_t n_tuner, int32_t n_groups,
                                            kareto_grid **out) {
  if (!ctx || !out) return KARETO_E_INVALID;
  *out = nullptr;
  ctx->err.clear();
  if (n_groups < 1 || n_groups > 1024) return kareto::fail(ctx, KARETO_E_INVALID, "n_groups must be in [1, 1024]");
  cudaSetDevice(ctx->device);
  kareto_grid *g = new kareto_grid();
  g->ctx = ctx;
  g->n = n_cfg;
  g->prep = new kareto::GridPrep();
  const bool cfg_shard = ctx->world > 1 || ctx->nccl;
  kareto_status s = kareto::prep_grid(ctx, cfg, n_cfg, ttl_ms, n_tuner, n_groups, cfg_shard, *g->prep);
  if (s == KARETO_OK && n_cfg > 0) {
    const std::string keep = ctx->err;  // a line-key range problem only matters if pruning is asked for
    g->lw_ok = kareto::pareto_line_widths(ctx, cfg, n_cfg, g->lw, &g->lw_err) == KARETO_OK;
    ctx->err = keep;
    cudaError_t e = cudaMallocFromPoolAsync((void **)&g->dall, sizeof(kareto_config) * n_cfg, ctx->pool, ctx->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(g->dall, cfg, sizeof(kareto_config) * n_cfg, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      s = kareto::fail(ctx, KARETO_E_OOM, "grid upload: %s", cudaGetErrorString(e));
    }
  } else if (s == KARETO_OK) {
    g->lw_ok = true;
    s = kareto::sync(ctx, "grid_create");
  }
  if (s != KARETO_OK) {
    kareto_grid_free(g);
    return s;
  }
  *out = g;
  return KARETO_OK;
}

extern "C" void kareto_grid_free(kareto_grid *g) {
  if (!g) return;
  if (g->dall) cudaFreeAsync(g->dall, g->ctx->stream);
  for (int a = 0; a < 3; a++) {
    if (g->lkey[a]) cudaFreeAsync(g->lkey[a], g->ctx->stream);
    if (g->lidx[a]) cudaFreeAsync(g->lidx[a], g->ctx->stream);
  }
  delete g->prep;  // its device buffers free on the context stream
  delete g->prep_whole;
  cudaStreamSynchronize(g->ctx->stream);
  (void)cudaGetLastError();
  delete g;
}

extern "C" kareto_status kareto_eval_grid_prepared(kareto_ctx *ctx, const kareto_trace *tr, const kareto_grid *grid,
                                                   const kareto_model *model, kareto_counts *counts_out,
                                                   double *obj_out, int32_t outputs_on_device) {
  if (!ctx || !tr || !grid) return KARETO_E_INVALID;
  ctx->err.clear();
  if (grid->ctx != ctx) return kareto::fail(ctx, KARETO_E_INVALID, "grid belongs to another context");
  cudaSetDevice(ctx->device);
  kareto_status s;
  if (grid->prep->cfg_shard && tr->sharded) {
    // a time-sharded trace evaluates the whole grid on every rank: the grid's configuration
    // shard does not apply; the unsharded split is derived once (from the device copy) and kept
    kareto_grid *g = const_cast<kareto_grid *>(grid);
    s = KARETO_OK;
    if (!g->prep_whole) {
      std::vector<kareto_config> h(grid->n);
      if (grid->n > 0) cudaMemcpy(h.data(), grid->dall, sizeof(kareto_config) * grid->n, cudaMemcpyDeviceToHost);
      const kareto::GridPrep &P = *grid->prep;
      g->prep_whole = new kareto::GridPrep();
      s = kareto::prep_grid(ctx, h.data(), grid->n, P.n_tuner ? P.rows.data() : nullptr, P.n_tuner, P.G, false,
                            *g->prep_whole);
      if (s != KARETO_OK) {
        delete g->prep_whole;
        g->prep_whole = nullptr;
      }
    }
    if (s == KARETO_OK) s = kareto::run_eval(ctx, tr, *g->prep_whole, model, counts_out, obj_out, outputs_on_device);
  } else {
    s = kareto::run_eval(ctx, tr, *grid->prep, model, counts_out, obj_out, outputs_on_device);
  }
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

extern "C" kareto_status kareto_shard_bounds(const kareto_config *cfg, int64_t n, const uint32_t *ttl_ms,
                                             int32_t n_tuner, int32_t n_groups, int32_t world, int64_t *bounds) {
  if (n < 0 || (n > 0 && !cfg) || world < 1 || n_groups < 1 || n_tuner < 0 || (n_tuner > 0 && !ttl_ms) || !bounds)
    return KARETO_E_INVALID;
  std::vector<uint32_t> rows;
  if (n_tuner == 0) rows.assign((size_t)n_groups, KARETO_TTL_INF);
  else rows.assign(ttl_ms, ttl_ms + (size_t)n_tuner * n_groups);
  for (int64_t i = 0; i < n; i++)
    if (n_tuner > 0 && cfg[i].tuner >= n_tuner) return KARETO_E_INVALID;
  kareto::shard_bounds(cfg, n, rows.data(), n_tuner, n_groups, world, bounds);
  return KARETO_OK;
}

extern "C" kareto_status kareto_shard_range(int64_t n, int32_t rank, int32_t world, int64_t *lo, int64_t *hi) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return KARETO_E_INVALID;
  kareto::shard_range(n, rank, world, *lo, *hi);
  return KARETO_OK;
}

extern "C" kareto_status kareto_eval_grid(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg,
                                          int64_t n_cfg, const uint32_t *ttl_ms, int32_t n_tuner,
                                          const kareto_model *model, kareto_counts *counts_out, double *obj_out,
                                          int32_t outputs_on_device) {
  if (!ctx || !tr) return KARETO_E_INVALID;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::eval(ctx, tr, cfg, n_cfg, ttl_ms, n_tuner, model, counts_out, obj_out, outputs_on_device);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

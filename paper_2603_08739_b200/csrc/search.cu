// search.cu -- row f1: the exact 3-D hypervolume and Alg. 1 "Adaptive Pareto
// Exploration" as a native driver over kareto_eval_grid / kareto_pareto.
//
// Hypervolume (R41), B200 design: HSO slicing along the third objective.  With the m
// selected points in (x, y)-lexicographic order and z-ranks r_i, slab k (between the k-th and
// (k+1)-th smallest z) has area
//     A_k = sum_{i : r_i <= k} (ref_x - x_i) * (ymin_{<i} - min(ymin_{<i}, y_i)),
// ymin_{<i} = min(ref_y, min{ y_j : j < i, r_j <= k }) -- the staircase swept in x.  One CTA per
// slab streams the x-ordered points (L2-resident: 24 B each) with a block-wide exclusive
// min-scan carried across chunks; HV = sum_k A_k (z_(k+1) - z_(k)), z_(m) = ref_z, reduced by
// CUB.  O(m^2) work for a frontier of m points, no shared-memory size limit.
//
// Search driver: host C++ over the library's own calls; each round's candidates go to the
// GPU in one kareto_eval_grid call (sharded over ranks when world > 1), the decisions of
// l.10-19 are taken on the returned fp64 objectives (bit-identical to the oracle's, so the
// evaluated set is identical), and the final frontier comes from kareto_pareto.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <set>
#include <vector>

#include "internal.cuh"

namespace kareto {

constexpr int HV_THREADS = 256;

__global__ void k_hv_gather(const double *__restrict__ obj, const uint32_t *__restrict__ sel, int m,
                            double rx, double ry, double rz, double *__restrict__ x, double *__restrict__ y,
                            double *__restrict__ z, uint32_t *__restrict__ idx, unsigned long long *__restrict__ bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const uint32_t s = sel[i];
    const double a = obj[3 * (size_t)s], b = obj[3 * (size_t)s + 1], c = obj[3 * (size_t)s + 2];
    x[i] = a;
    y[i] = b;
    z[i] = c;
    idx[i] = (uint32_t)i;
    if (!(a < rx && b < ry && c < rz)) atomicMin(bad, (unsigned long long)s);
  }
}

// zrank of every point from the z order
__global__ void k_hv_zrank(const uint32_t *__restrict__ zord, int m, uint32_t *__restrict__ zrank) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) zrank[zord[k]] = (uint32_t)k;
}

// points in (x, y) order: X, Y, rank
__global__ void k_hv_xorder(const uint32_t *__restrict__ xord, const double *__restrict__ x,
                            const double *__restrict__ y, const uint32_t *__restrict__ zrank, int m,
                            double *__restrict__ X, double *__restrict__ Y, uint32_t *__restrict__ Rk) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const uint32_t p = xord[i];
    X[i] = x[p];
    Y[i] = y[p];
    Rk[i] = zrank[p];
  }
}

struct MinOpD {
  __device__ __forceinline__ double operator()(double a, double b) const { return b < a ? b : a; }
};

__global__ void __launch_bounds__(HV_THREADS) k_hv_slabs(const double *__restrict__ X, const double *__restrict__ Y,
                                                          const uint32_t *__restrict__ Rk,
                                                          const double *__restrict__ zs, int m, double rx,
                                                          double ry, double rz, double *__restrict__ vol) {
  typedef cub::BlockScan<double, HV_THREADS> Scan;
  typedef cub::BlockReduce<double, HV_THREADS> Red;
  __shared__ typename Scan::TempStorage ts;
  __shared__ typename Red::TempStorage tr;
  __shared__ double carry_s;
  for (int k = blockIdx.x; k < m; k += gridDim.x) {
    const double z0 = zs[k], z1 = k + 1 < m ? zs[k + 1] : rz;
    if (!(z1 > z0)) {  // zero-thickness slab (tied z)
      if (threadIdx.x == 0) vol[k] = 0.0;
      continue;
    }
    double carry = ry, area = 0.0;
    for (int base = 0; base < m; base += HV_THREADS) {
      const int i = base + threadIdx.x;
      const bool in = i < m && Rk[i] <= (uint32_t)k;
      const double yv = in ? Y[i] : INFINITY;
      double excl;
      Scan(ts).ExclusiveScan(yv, excl, (double)INFINITY, MinOpD());
      const double pm = excl < carry ? excl : carry;  // running minimum before point i
      if (in && yv < pm) area += (rx - X[i]) * (pm - yv);
      // the chunk's minimum is the inclusive value of the last lane
      if (threadIdx.x == HV_THREADS - 1) carry_s = yv < pm ? yv : pm;
      __syncthreads();
      carry = carry_s;
      __syncthreads();
    }
    const double A = Red(tr).Sum(area);
    if (threadIdx.x == 0) vol[k] = A * (z1 - z0);
    __syncthreads();
  }
}

template <typename F>
static kareto_status cub_run(kareto_ctx *ctx, DBuf<uint8_t> &tmp, F &&f) {
  size_t bytes = 0;
  KCUDA(ctx, f((void *)nullptr, bytes));
  if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
  size_t b2 = tmp.n;
  KCUDA(ctx, f((void *)tmp.p, b2));
  return KARETO_OK;
}

static kareto_status hypervolume(kareto_ctx *ctx, const double *obj, const uint8_t *mask, int64_t n,
                                 const double ref[3], double *hv_out, int on_dev) {
  if (n < 0 || !ref || !hv_out || (n > 0 && !obj)) return fail(ctx, KARETO_E_INVALID, "hypervolume: bad arguments");
  if (n >= (int64_t)1 << 31) return fail(ctx, KARETO_E_INVALID, "hypervolume: n >= 2^31");
  *hv_out = 0.0;
  if (n == 0) return KARETO_OK;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  DBuf<double> fown;
  DBuf<uint8_t> mown, tmp;
  const double *f = obj;
  const uint8_t *mk = mask;
  if (!on_dev) {
    KTRY(fown.alloc(ctx, 3 * n));
    KCUDA(ctx, cudaMemcpyAsync(fown.p, obj, 24 * n, cudaMemcpyHostToDevice, st));
    f = fown.p;
    if (mask) {
      KTRY(mown.alloc(ctx, n));
      KCUDA(ctx, cudaMemcpyAsync(mown.p, mask, n, cudaMemcpyHostToDevice, st));
      mk = mown.p;
    }
  }
  // selected indices
  DBuf<uint32_t> sel;
  DBuf<int> m_dev;
  KTRY(sel.alloc(ctx, n)); KTRY(m_dev.alloc(ctx, 1));
  int m = (int)n;
  {
    Pass ps(ctx, "F1_hv_select", 0, 1);
    cub::CountingInputIterator<uint32_t> it(0);
    if (mk) {
      KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceSelect::Flagged(t, b, it, mk, sel.p, m_dev.p, (int)n, st);
      }));
      KCUDA(ctx, cudaMemcpyAsync(&m, m_dev.p, 4, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
    } else {
      KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceSelect::Flagged(t, b, it, cub::ConstantInputIterator<uint8_t>(1), sel.p, m_dev.p,
                                          (int)n, st);
      }));
    }
  }
  if (m == 0) return KARETO_OK;
  DBuf<double> x, y, z, xs, ys, zs, X, Y, vol, hv;
  DBuf<uint32_t> i0, i1, i2, zrank, Rk;
  DBuf<unsigned long long> bad;
  for (DBuf<double> *b : {&x, &y, &z, &xs, &ys, &zs, &X, &Y, &vol}) KTRY(b->alloc(ctx, m));
  for (DBuf<uint32_t> *b : {&i0, &i1, &i2, &zrank, &Rk}) KTRY(b->alloc(ctx, m));
  KTRY(bad.alloc(ctx, 1)); KTRY(hv.alloc(ctx, 1));
  KCUDA(ctx, cudaMemsetAsync(bad.p, 0xFF, 8, st));
  {
    Pass ps(ctx, "F1_hv_prepare", 1, 3);
    k_hv_gather<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(f, sel.p, m, ref[0], ref[1], ref[2], x.p, y.p, z.p,
                                                             i0.p, bad.p);
    unsigned long long hbad = 0;
    KCUDA(ctx, cudaMemcpyAsync(&hbad, bad.p, 8, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    if (hbad != ~0ull)
      return fail(ctx, KARETO_E_INVALID, "hypervolume: reference point not strictly worse than point %llu", hbad);
    // z order (stable) -> ranks
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, z.p, zs.p, i0.p, i1.p, m, 0, 64, st);
    }));
    k_hv_zrank<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(i1.p, m, zrank.p);
    // (x, y) lexicographic: stable sort by y, then by x
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, y.p, ys.p, i0.p, i1.p, m, 0, 64, st);
    }));
    k_hv_xorder<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(i1.p, x.p, y.p, zrank.p, m, X.p, Y.p, Rk.p);
    // X currently in y order: sort (x of y-ordered) keeping the y-order permutation
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, X.p, xs.p, i1.p, i2.p, m, 0, 64, st);
    }));
    k_hv_xorder<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(i2.p, x.p, y.p, zrank.p, m, X.p, Y.p, Rk.p);
  }
  {
    Pass ps(ctx, "F1_hv_slabs", 1, 1);
    const int grid = m < 64 * sms ? m : 64 * sms;
    k_hv_slabs<<<grid, HV_THREADS, 0, st>>>(X.p, Y.p, Rk.p, zs.p, m, ref[0], ref[1], ref[2], vol.p);
  }
  {
    Pass ps(ctx, "F1_hv_sum", 0, 1);
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) { return cub::DeviceReduce::Sum(t, b, vol.p, hv.p, m, st); }));
  }
  KCUDA(ctx, cudaMemcpyAsync(hv_out, hv.p, 8, cudaMemcpyDeviceToHost, st));
  return sync(ctx, "hypervolume");
}

// ------------------------------------------------------------------ Alg. 1 driver
static double rel_delta(double a, double b) {  // R36
  return std::fabs(a - b) / std::fmax(std::fmax(std::fabs(a), std::fabs(b)), 1e-9);
}

typedef std::pair<int64_t, int64_t> DT;

static kareto_status search(kareto_ctx *ctx, const kareto_trace *tr, const kareto_search_params *p,
                            const kareto_model *model, kareto_search_point *out, int64_t cap, int64_t *n_out,
                            int32_t *truncated) {
  if (!tr || !p || !model || !n_out || !truncated || cap < 0 || (cap > 0 && !out))
    return fail(ctx, KARETO_E_INVALID, "search: bad arguments");
  if (p->d_step < 1 || p->t_step < 1 || p->d_min < 0 || p->t_min < 0 || p->d_max < p->d_min || p->t_max < p->t_min)
    return fail(ctx, KARETO_E_INVALID, "search: bad DRAM / TTL ranges");
  if (p->t_max > (int64_t)(0xFFFFFFFEu / 1000)) return fail(ctx, KARETO_E_INVALID, "search: TTL above 2^32 ms");
  if (!(p->hbm_gb >= 0) || !std::isfinite(p->hbm_gb) || !(p->tau_e >= 0) || !(p->tau_perf >= 0) ||
      !(p->tau_cost >= 0) || p->policy < 0 || p->policy > 2 || p->max_rounds < 0 || model->block_bytes == 0 ||
      p->expand_ttl < 0 || p->expand_ttl > 1)
    return fail(ctx, KARETO_E_INVALID, "search: bad thresholds / policy / model");
  const int G = tr->K + 1;
  const uint64_t Bb = model->block_bytes;
  const uint64_t hbm = (uint64_t)(p->hbm_gb * 1e9) / Bb;
  *n_out = 0;
  *truncated = 0;
  std::map<DT, std::array<double, 3>> S;
  std::vector<kareto_search_point> log;
  std::vector<DT> C;
  for (int64_t d = p->d_min; d <= p->d_max; d += p->d_step)
    for (int64_t t = p->t_min; t <= p->t_max; t += p->t_step) C.push_back({d, t});
  std::sort(C.begin(), C.end());
  int rnd = 0;
  while (!C.empty()) {
    if ((int64_t)(S.size() + C.size()) > cap || (p->max_rounds && rnd >= p->max_rounds)) {
      *truncated = 1;  // R40
      break;
    }
    // l.5-8: one batched evaluation of the round's candidates
    std::vector<int64_t> ts;
    for (auto &c : C) ts.push_back(c.second);
    std::sort(ts.begin(), ts.end());
    ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
    std::vector<uint32_t> rows((size_t)ts.size() * G);
    for (size_t r = 0; r < ts.size(); r++)
      for (int g = 0; g < G; g++) rows[r * G + g] = (uint32_t)(ts[r] * 1000);
    std::vector<kareto_config> cf(C.size());
    for (size_t i = 0; i < C.size(); i++) {
      kareto_config &c = cf[i];
      memset(&c, 0, sizeof(c));
      c.cap[0] = hbm;
      c.cap[1] = (uint64_t)C[i].first * 1000000000ull / Bb;
      c.cap[2] = KARETO_INF;
      c.policy = (uint8_t)p->policy;
      c.tuner = (uint16_t)(std::lower_bound(ts.begin(), ts.end(), C[i].second) - ts.begin());
    }
    if (ts.size() > 65535) return fail(ctx, KARETO_E_INVALID, "search: more than 65535 TTL values in a round");
    std::vector<double> F(3 * C.size());
    KTRY(kareto_eval_grid(ctx, tr, cf.data(), (int64_t)cf.size(), rows.data(), (int32_t)ts.size(), model, nullptr,
                          F.data(), 0));
    for (size_t i = 0; i < C.size(); i++) {
      S[C[i]] = {F[3 * i], F[3 * i + 1], F[3 * i + 2]};
      kareto_search_point q;
      memset(&q, 0, sizeof(q));
      q.d_gb = C[i].first;
      q.t_s = C[i].second;
      q.obj[0] = F[3 * i];
      q.obj[1] = F[3 * i + 1];
      q.obj[2] = F[3 * i + 2];
      q.round = rnd;
      log.push_back(q);
    }
    rnd++;
    std::set<DT> cand;  // l.9
    // l.10-14: DRAM expansion at the lowest TTL column (R37)
    int64_t dmax = -1;
    for (auto &kv : S)
      if (kv.first.second == p->t_min) dmax = std::max(dmax, kv.first.first);
    if (dmax >= 0) {
      auto lo = S.find({dmax - p->d_step, p->t_min});
      if (lo != S.end() && rel_delta(lo->second[0], S[{dmax, p->t_min}][0]) > p->tau_e)
        for (int64_t t = p->t_min; t <= p->t_max; t += p->t_step) cand.insert({dmax + p->d_step, t});
    }
    // R55 (extension, off by default): the same test along the TTL axis at the lowest DRAM row;
    // the new row spans the initial DRAM range; TTLs stay below 2^32 ms
    if (p->expand_ttl) {
      int64_t tmax = -1;
      for (auto &kv : S)
        if (kv.first.first == p->d_min) tmax = std::max(tmax, kv.first.second);
      if (tmax >= 0 && tmax + p->t_step <= (int64_t)(0xFFFFFFFEu / 1000)) {
        auto lo = S.find({p->d_min, tmax - p->t_step});
        if (lo != S.end() && rel_delta(lo->second[0], S[{p->d_min, tmax}][0]) > p->tau_e)
          for (int64_t d = p->d_min; d <= p->d_max; d += p->d_step) cand.insert({d, tmax + p->t_step});
      }
    }
    // l.15-19: refinement of adjacent pairs (R38, R39)
    std::map<int64_t, std::vector<int64_t>> by_t, by_d;
    for (auto &kv : S) {
      by_t[kv.first.second].push_back(kv.first.first);
      by_d[kv.first.first].push_back(kv.first.second);
    }
    auto consider = [&](DT a, DT b) {
      const auto &fa = S[a], &fb = S[b];
      if ((rel_delta(fa[0], fb[0]) > p->tau_perf || rel_delta(fa[1], fb[1]) > p->tau_perf) &&
          rel_delta(fa[2], fb[2]) > p->tau_cost) {
        DT mid{(a.first + b.first) / 2, (a.second + b.second) / 2};
        if (mid != a && mid != b) cand.insert(mid);
      }
    };
    for (auto &kv : by_t) {
      auto &ds = kv.second;  // ascending (map order)
      for (size_t i = 0; i + 1 < ds.size(); i++) consider({ds[i], kv.first}, {ds[i + 1], kv.first});
    }
    for (auto &kv : by_d) {
      auto &tv = kv.second;
      for (size_t i = 0; i + 1 < tv.size(); i++) consider({kv.first, tv[i]}, {kv.first, tv[i + 1]});
    }
    C.clear();
    for (auto &c : cand)
      if (!S.count(c)) C.push_back(c);  // std::set: ascending (d, t)
  }
  // l.22: ParetoFilter(P)
  const int64_t n = (int64_t)log.size();
  if (n > 0) {
    std::vector<double> F(3 * n);
    std::vector<kareto_config> cf(n);
    std::vector<uint8_t> stv(n);
    memset(cf.data(), 0, sizeof(kareto_config) * n);
    for (int64_t i = 0; i < n; i++)
      for (int a = 0; a < 3; a++) F[3 * i + a] = log[i].obj[a];
    KTRY(kareto_pareto(ctx, F.data(), cf.data(), n, nullptr, stv.data(), nullptr, 0));
    for (int64_t i = 0; i < n; i++) log[i].status = stv[i];
    memcpy(out, log.data(), sizeof(kareto_search_point) * n);
  }
  *n_out = n;
  return KARETO_OK;
}

}  // namespace kareto

extern "C" kareto_status kareto_hypervolume(kareto_ctx *ctx, const double *obj, const uint8_t *mask, int64_t n,
                                            const double ref[3], double *hv_out, int32_t on_device) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::hypervolume(ctx, obj, mask, n, ref, hv_out, on_device);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

extern "C" kareto_status kareto_search(kareto_ctx *ctx, const kareto_trace *tr, const kareto_search_params *params,
                                       const kareto_model *model, kareto_search_point *out, int64_t cap,
                                       int64_t *n_out, int32_t *truncated) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  return kareto::search(ctx, tr, params, model, out, cap, n_out, truncated);
}

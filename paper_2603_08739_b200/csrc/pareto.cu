// pareto.cu -- kareto_pareto: rows a9 (K8a diminishing-return pruning, Alg. 1 expansion
// test P:555-559 / P:532, R34) and a10 (K8b non-dominance, R35).
//
// K8a: per capacity axis a, configurations are sorted by (line key, axis index a, index)
// with one 64-bit radix key; a line's first step with rel <= tau_e stops it and every
// later point of the line is pruned (segmented exclusive OR-scan).
// K8b: survivors sorted by f1; a point can only be dominated by points whose f1 is <= its
// own, so each thread scans that prefix (smem tiles) and stops at its first dominator.
// All decisions are exact IEEE comparisons: results are independent of ordering.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace kareto {

// Line key of axis a, packed with the bit widths the configurations actually use (w[0..2]: axis
// index widths, w[3] tuner, w[4] medium, w[5] policy): low to high, axis[a] | axis[o2] | axis[o1]
// | tuner | medium | policy.  Sorting only the used bits groups each line and orders it by
// axis[a]; the order of the lines does not matter (the scan restarts per line).
struct LineWidths {
  int w[6];
};
__global__ void k_line_keys(const kareto_config *__restrict__ cfg, int64_t n, int a, LineWidths lw,
                            uint64_t *__restrict__ key, uint32_t *__restrict__ idx) {
  const int o1 = (a + 1) % 3, o2 = (a + 2) % 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const kareto_config c = cfg[i];
    uint64_t k = c.policy;
    k = (k << lw.w[4]) | c.medium;
    k = (k << lw.w[3]) | c.tuner;
    k = (k << lw.w[o1]) | (uint32_t)c.axis[o1];
    k = (k << lw.w[o2]) | (uint32_t)c.axis[o2];
    k = (k << lw.w[a]) | (uint32_t)c.axis[a];
    key[i] = k;
    idx[i] = (uint32_t)i;
  }
}

__global__ void k_line_stop(const uint64_t *__restrict__ key, const uint32_t *__restrict__ idx, int64_t n, int wa,
                            const double *__restrict__ f, double tau_e, uint64_t *__restrict__ line,
                            uint8_t *__restrict__ stop) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t li = key[i] >> wa;
    line[i] = li;
    uint8_t s = 0;
    if (i > 0 && (key[i - 1] >> wa) == li) {
      double p = f[3 * (size_t)idx[i - 1]], q = f[3 * (size_t)idx[i]];
      double ap = p < 0 ? -p : p, aq = q < 0 ? -q : q;
      double den = ap > aq ? ap : aq;
      den = den > 1e-9 ? den : 1e-9;
      double rel = (p - q) / den;
      s = rel <= tau_e ? 1 : 0;
    }
    stop[i] = s;
  }
}

// Short lines (at most 2^wa points): the segmented exclusive OR-scan done in place -- each point
// walks back through its line to the first earlier stop (or the line start) and marks itself
__global__ void k_line_prune(const uint64_t *__restrict__ key, const uint32_t *__restrict__ idx, int64_t n, int wa,
                             const uint8_t *__restrict__ stop, uint8_t *__restrict__ pruned) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t li = key[i] >> wa;
    for (int64_t k = i - 1; k >= 0 && (key[k] >> wa) == li; k--)
      if (stop[k]) {
        pruned[idx[i]] = 1;
        break;
      }
  }
}

__global__ void k_mark_pruned(const uint8_t *__restrict__ excl, const uint32_t *__restrict__ idx, int64_t n,
                              uint8_t *__restrict__ pruned) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (excl[i]) pruned[idx[i]] = 1;
}

__global__ void k_survivor_flags(const uint8_t *__restrict__ pruned, int64_t n, uint8_t *__restrict__ keep,
                                 double *__restrict__ f1, const double *__restrict__ f, uint32_t *__restrict__ idx,
                                 int *__restrict__ m_all) {
  if (m_all && blockIdx.x == 0 && threadIdx.x == 0) *m_all = (int)n;  // no pruning: every point survives
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keep[i] = pruned[i] ? 0 : 1;
    f1[i] = f[3 * i];
    idx[i] = (uint32_t)i;
  }
}

constexpr int P_THREADS = 256;
constexpr int P_TILE = 512;

// survivors sorted by f1 (sidx): thread = one candidate x; scan candidates y with
// f1(y) <= f1(x) until a dominator is found.
__global__ void __launch_bounds__(P_THREADS) k_dominance(const uint32_t *__restrict__ sidx, const int *__restrict__ m_ptr,
                                                         const double *__restrict__ f, uint8_t *__restrict__ status,
                                                         unsigned long long *__restrict__ n_front) {
  __shared__ double tf[P_TILE][3];
  const int m = *m_ptr;
  const int a = blockIdx.x * P_THREADS + threadIdx.x;
  if ((int64_t)blockIdx.x * P_THREADS >= m) return;
  double x0 = 0, x1 = 0, x2 = 0;
  bool mine = a < m;
  if (mine) {
    const double *px = f + 3 * (size_t)sidx[a];
    x0 = px[0]; x1 = px[1]; x2 = px[2];
  }
  // CTA bound: the largest f1 among its candidates
  int last = (blockIdx.x + 1) * P_THREADS - 1;
  if (last >= m) last = m - 1;
  const double bound = f[3 * (size_t)sidx[last]];
  bool dom = false;
  for (int t0 = 0; t0 < m; t0 += P_TILE) {
    if (f[3 * (size_t)sidx[t0]] > bound) break;  // sorted: nothing later can dominate anyone here
    __syncthreads();
    for (int k = threadIdx.x; k < P_TILE; k += P_THREADS) {
      int b = t0 + k;
      if (b < m) {
        const double *py = f + 3 * (size_t)sidx[b];
        tf[k][0] = py[0]; tf[k][1] = py[1]; tf[k][2] = py[2];
      } else {
        tf[k][0] = 1.0 / 0.0; tf[k][1] = 0; tf[k][2] = 0;
      }
    }
    __syncthreads();
    if (mine && !dom) {
      for (int k = 0; k < P_TILE; k++) {
        double y0 = tf[k][0];
        if (y0 > x0) break;
        double y1 = tf[k][1], y2 = tf[k][2];
        if (y1 <= x1 && y2 <= x2 && (y0 < x0 || y1 < x1 || y2 < x2)) { dom = true; break; }
      }
    }
    if (__syncthreads_and(!mine || dom)) break;
  }
  if (mine) {
    status[sidx[a]] = dom ? 0 : 1;
    if (!dom) atomicAdd(n_front, 1ull);
  }
}

__global__ void k_status_pruned(const uint8_t *__restrict__ pruned, int64_t n, uint8_t *__restrict__ status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (pruned[i]) status[i] = 2;
}

struct MaxOp {
  __device__ __forceinline__ uint8_t operator()(uint8_t a, uint8_t b) const { return a > b ? a : b; }
};

template <typename F>
static kareto_status cub_tmp(kareto_ctx *ctx, DBuf<uint8_t> &tmp, F &&f) {
  size_t bytes = 0;
  KCUDA(ctx, f((void *)nullptr, bytes));
  if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
  size_t b2 = tmp.n;
  KCUDA(ctx, f((void *)tmp.p, b2));
  return KARETO_OK;
}

// Host checks of the line keys pruning builds (axis and key fields in range) and their bit widths.
kareto_status pareto_line_widths(kareto_ctx *ctx, const kareto_config *cfg, int64_t n, int *w, std::string *err) {
  uint32_t mx[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = 0; i < n; i++) {
    const kareto_config &c = cfg[i];
    for (int a = 0; a < 3; a++) {
      if (c.axis[a] < 0 || c.axis[a] > 65535) {
        char b[96];
        snprintf(b, sizeof(b), "config %lld: axis out of range", (long long)i);
        if (err) *err = b;
        return fail(ctx, KARETO_E_INVALID, "%s", b);
      }
      mx[a] |= (uint32_t)c.axis[a];
    }
    if (c.tuner > 1023 || c.medium > 15 || c.policy > 3) {
      char b[96];
      snprintf(b, sizeof(b), "config %lld: line key out of range", (long long)i);
      if (err) *err = b;
      return fail(ctx, KARETO_E_INVALID, "%s", b);
    }
    mx[3] |= c.tuner; mx[4] |= c.medium; mx[5] |= c.policy;
  }
  for (int k = 0; k < 6; k++) {  // bits needed by the OR of the values = bits of the maximum
    w[k] = 0;
    while (w[k] < 32 && (mx[k] >> w[k]) != 0) w[k]++;
  }
  return KARETO_OK;
}

// dcfg: device copy of the configurations (only read when pruning), lw: their line-key widths
static kareto_status pareto_run(kareto_ctx *ctx, const double *obj, const kareto_config *dcfg_in, const kareto_config *hcfg,
                                const LineWidths &lw, int64_t n, const kareto_prune *prune, uint8_t *status_out,
                                int64_t *n_frontier, int32_t on_dev, kareto_grid *grid = nullptr);

static kareto_status pareto(kareto_ctx *ctx, const double *obj, const kareto_config *cfg, int64_t n,
                            const kareto_prune *prune, uint8_t *status_out, int64_t *n_frontier, int32_t on_dev) {
  if (n < 0 || (n > 0 && (!obj || !status_out))) return fail(ctx, KARETO_E_INVALID, "bad arguments");
  if (n >= (int64_t)0x7FFFFFFF) return fail(ctx, KARETO_E_OVERFLOW, "too many configurations");
  const bool do_prune = prune && prune->enabled;
  LineWidths lw{};
  if (do_prune) {
    if (!cfg) return fail(ctx, KARETO_E_INVALID, "pruning needs the configurations");
    KTRY(pareto_line_widths(ctx, cfg, n, lw.w, nullptr));
  }
  return pareto_run(ctx, obj, nullptr, cfg, lw, n, prune, status_out, n_frontier, on_dev);
}

static kareto_status pareto_run(kareto_ctx *ctx, const double *obj, const kareto_config *dcfg_in, const kareto_config *hcfg,
                                const LineWidths &lw, int64_t n, const kareto_prune *prune, uint8_t *status_out,
                                int64_t *n_frontier, int32_t on_dev, kareto_grid *grid) {
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const bool do_prune = prune && prune->enabled;
  int key_bits = 0;
  for (int k = 0; k < 6; k++) key_bits += lw.w[k];
  if (key_bits == 0) key_bits = 1;
  if (n == 0) {
    if (n_frontier) *n_frontier = 0;
    return KARETO_OK;
  }
  DBuf<double> fown;
  const double *f = obj;
  if (!on_dev) {
    KTRY(fown.alloc(ctx, 3 * n));
    KCUDA(ctx, cudaMemcpyAsync(fown.p, obj, 24 * n, cudaMemcpyHostToDevice, st));
    f = fown.p;
  }
  DBuf<uint8_t> tmp, pruned, status;
  KTRY(pruned.alloc(ctx, n)); KTRY(pruned.zero());
  KTRY(status.alloc(ctx, n));
  if (do_prune) {
    DBuf<kareto_config> down;
    DBuf<uint64_t> key, key_s, line;
    DBuf<uint32_t> idx, idx_s;
    DBuf<uint8_t> stop, excl;
    KTRY(key.alloc(ctx, n)); KTRY(key_s.alloc(ctx, n)); KTRY(line.alloc(ctx, n));
    KTRY(idx.alloc(ctx, n)); KTRY(idx_s.alloc(ctx, n)); KTRY(stop.alloc(ctx, n)); KTRY(excl.alloc(ctx, n));
    const kareto_config *dcfg = dcfg_in;
    if (!dcfg) {
      KTRY(down.alloc(ctx, n));
      KCUDA(ctx, cudaMemcpyAsync(down.p, hcfg, sizeof(kareto_config) * n, cudaMemcpyHostToDevice, st));
      dcfg = down.p;
    }
    for (int a = 0; a < 3; a++) {
      // a prepared grid sorts its lines once (first selection) and keeps (key, permutation)
      const bool cached = grid && grid->lkey[a];
      uint64_t *ks = cached ? grid->lkey[a] : key_s.p;
      uint32_t *is = cached ? grid->lidx[a] : idx_s.p;
      if (!cached) {
        {
          Pass ps(ctx, "K8a_line_keys", 1, 1);
          k_line_keys<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(dcfg, n, a, lw, key.p, idx.p);
        }
        Pass ps(ctx, "K8a_sort_lines", 0, 1);
        KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
          return cub::DeviceRadixSort::SortPairs(t, b, key.p, key_s.p, idx.p, idx_s.p, (int)n, 0, key_bits, st);
        }));
        if (grid) {  // the sorted copies move to the grid (fresh ones for the next axis)
          grid->lkey[a] = key_s.detach();
          grid->lidx[a] = idx_s.detach();
          KTRY(key_s.alloc(ctx, n));
          KTRY(idx_s.alloc(ctx, n));
        }
      }
      {
        Pass ps(ctx, "K8a_line_stop", 1, 2);
        k_line_stop<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(ks, is, n, lw.w[a], f, prune->tau_e, line.p, stop.p);
        if (lw.w[a] <= 8) {  // lines of <= 256 points: walk back instead of a segmented scan
          k_line_prune<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(ks, is, n, lw.w[a], stop.p, pruned.p);
        } else {
          KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
            return cub::DeviceScan::ExclusiveScanByKey(t, b, line.p, stop.p, excl.p, MaxOp(), (uint8_t)0, (int)n,
                                                       cub::Equality(), st);
          }));
          k_mark_pruned<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(excl.p, is, n, pruned.p);
        }
      }
    }
  }
  // K8b
  DBuf<unsigned long long> nf;
  KTRY(nf.alloc(ctx, 1)); KTRY(nf.zero());
  {
    DBuf<uint8_t> keep;
    DBuf<double> f1, f1c, f1s;
    DBuf<uint32_t> idx, idxc, idxs;
    DBuf<int> m_dev;
    KTRY(keep.alloc(ctx, n)); KTRY(f1.alloc(ctx, n)); KTRY(f1c.alloc(ctx, n)); KTRY(f1s.alloc(ctx, n));
    KTRY(idx.alloc(ctx, n)); KTRY(idxc.alloc(ctx, n)); KTRY(idxs.alloc(ctx, n)); KTRY(m_dev.alloc(ctx, 1));
    if (!do_prune) {  // every configuration survives: no compaction, no round trip for the count
      Pass ps(ctx, "K8b_compact_sort", 0, 2);
      k_survivor_flags<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(pruned.p, n, keep.p, f1.p, f, idx.p, m_dev.p);
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, f1.p, f1s.p, idx.p, idxs.p, (int)n, 0, 64, st);
      }));
      ctx->own_launches += 1;
    } else {
      Pass ps(ctx, "K8b_compact_sort", 0, 3);
      k_survivor_flags<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(pruned.p, n, keep.p, f1.p, f, idx.p, nullptr);
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceSelect::Flagged(t, b, f1.p, keep.p, f1c.p, m_dev.p, (int)n, st);
      }));
      KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceSelect::Flagged(t, b, idx.p, keep.p, idxc.p, m_dev.p, (int)n, st);
      }));
      int m = 0;
      KCUDA(ctx, cudaMemcpyAsync(&m, m_dev.p, 4, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      if (m > 0) {
        KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
          return cub::DeviceRadixSort::SortPairs(t, b, f1c.p, f1s.p, idxc.p, idxs.p, m, 0, 64, st);
        }));
      }
      ctx->own_launches += 1;
    }
    {
      Pass ps(ctx, "K8b_dominance", 1, 2);
      k_dominance<<<grid_for(n, P_THREADS), P_THREADS, 0, st>>>(idxs.p, m_dev.p, f, status.p, nf.p);
      k_status_pruned<<<grid_for(n, 256, 4 * sms), 256, 0, st>>>(pruned.p, n, status.p);
    }
  }
  unsigned long long hnf = 0;
  KCUDA(ctx, cudaMemcpyAsync(status_out, status.p, n, on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaMemcpyAsync(&hnf, nf.p, 8, cudaMemcpyDeviceToHost, st));
  KTRY(sync(ctx, "pareto"));
  if (n_frontier) *n_frontier = (int64_t)hnf;
  return KARETO_OK;
}

kareto_status pareto_grid(kareto_ctx *ctx, const double *obj, kareto_grid *g, const kareto_prune *prune,
                          uint8_t *status_out, int64_t *n_frontier, int32_t on_dev) {
  const int64_t n = g->n;
  if (n > 0 && (!obj || !status_out)) return fail(ctx, KARETO_E_INVALID, "bad arguments");
  if (n >= (int64_t)0x7FFFFFFF) return fail(ctx, KARETO_E_OVERFLOW, "too many configurations");
  LineWidths lw{};
  if (prune && prune->enabled) {
    if (!g->lw_ok) return fail(ctx, KARETO_E_INVALID, "%s", g->lw_err.c_str());
    for (int k = 0; k < 6; k++) lw.w[k] = g->lw[k];
  }
  return pareto_run(ctx, obj, g->dall, nullptr, lw, n, prune, status_out, n_frontier, on_dev, g);
}

}  // namespace kareto

extern "C" kareto_status kareto_pareto(kareto_ctx *ctx, const double *obj, const kareto_config *cfg, int64_t n,
                                       const kareto_prune *prune, uint8_t *status_out, int64_t *n_frontier,
                                       int32_t on_device) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::pareto(ctx, obj, cfg, n, prune, status_out, n_frontier, on_device);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

extern "C" kareto_status kareto_pareto_prepared(kareto_ctx *ctx, const double *obj, const kareto_grid *grid,
                                                const kareto_prune *prune, uint8_t *status_out, int64_t *n_frontier,
                                                int32_t on_device) {
  if (!ctx || !grid) return KARETO_E_INVALID;
  ctx->err.clear();
  if (grid->ctx != ctx) return kareto::fail(ctx, KARETO_E_INVALID, "grid belongs to another context");
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::pareto_grid(ctx, obj, const_cast<kareto_grid *>(grid), prune, status_out, n_frontier,
                                        on_device);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

// queue.cu -- row f3: queue-coupled disk prefetch and per-request TTFT distributions (PAPER.md
// Obs. 2 and 4; P99 TTFT constraints), R49-R53.
//
// For every stack-eligible LRU configuration, the requests are replayed through an FCFS queue
// over I identical instances: a request's disk-resident prefix blocks are prefetched during its
// queue wait only ("disk-based KV reloading exclusively during queuing time"), so the
// realised hit prefix -- and with it prefill time, TTFT and the instance's busy time -- depends
// on the wait, which depends on every earlier request.
//
// B200 design, per wave of configurations sized to free HBM:
//   1. k_queue_counts -- data-parallel over (request, configuration): each request's tier hits
//      from its accesses' pre-request LRU depths and reuse intervals (a CTA per request, threads
//      over configurations, broadcast loads of the accesses), stored [request][configuration];
//   2. k_queue -- the sequential part only: one thread per configuration walks the requests,
//      reading its counts coalesced, the instances' free times in shared memory; writes each
//      request's TTFT to a per-configuration row;
//   3. the exact nearest-rank P99 from a CUB segmented sort of the rows.
// Compiled with -fmad=false: the fp64 sequence is the oracle's, term by term (R33).
#include <cub/cub.cuh>

#include <vector>

#include "internal.cuh"
#include "replay.cuh"

namespace kareto {

__device__ __forceinline__ double qmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double qmin(double a, double b) { return a < b ? a : b; }

// R49, data-parallel over (request, configuration): a CTA per request, threads over the wave's
// configurations; every thread scans the request's accesses (the same addresses across the
// CTA: broadcast loads) and stores (h1, h2, h3) at [request][configuration].
__global__ void __launch_bounds__(128) k_queue_counts(const uint32_t *__restrict__ s,
                                                      const uint32_t *__restrict__ depth,
                                                      const uint32_t *__restrict__ delta,
                                                      const uint16_t *__restrict__ grp, int64_t R,
                                                      const kareto_config *__restrict__ cfg,
                                                      const uint32_t *__restrict__ rows, int n_tuner, int G,
                                                      int64_t nw, uint4 *__restrict__ cnt) {
  for (int64_t r = blockIdx.x; r < R; r += gridDim.x) {
    const uint32_t s0 = s[r], s1 = s[r + 1];
    const uint16_t g = grp[r];
    for (int64_t c = threadIdx.x; c < nw; c += blockDim.x) {
      const kareto_config cf = cfg[c];
      const bool ttl = cf.cap[2] == KARETO_INF;
      const uint64_t c1 = cf.cap[0], c12 = cf.cap[0] + cf.cap[1];
      const uint64_t C = ttl ? c12 : c12 + cf.cap[2];
      const uint32_t tg = rows[(size_t)(n_tuner > 0 ? cf.tuner : 0) * G + g];
      uint32_t h1 = 0, h2 = 0, h3 = 0;
#pragma unroll 4
      for (uint32_t j = s0; j < s1; j++) {
        const uint32_t dj = depth[j];
        if (dj == kNone) continue;
        if (dj <= c1) h1++;
        else if (dj <= c12) h2++;
        else if ((ttl || dj <= C) && delta[j] <= tg) h3++;
      }
      cnt[(size_t)r * nw + c] = make_uint4(h1, h2, h3, 0);
    }
  }
}

// R50-R53: one thread per configuration walks the requests; the instances' free times live in
// shared memory (SMEM) or in an [instance][configuration] global array.
template <bool SMEM>
__global__ void __launch_bounds__(32) k_queue(const int64_t *__restrict__ arr, const uint32_t *__restrict__ inlen,
                                              const uint32_t *__restrict__ outlen, int64_t R,
                                              const kareto_config *__restrict__ cfg, int64_t n,
                                              const uint4 *__restrict__ cnt, const kareto_model m, uint64_t span_ms,
                                              uint64_t LO, double *__restrict__ Fg, double *__restrict__ ttft,
                                              kareto_queue_result *__restrict__ out) {
  extern __shared__ double Fs[];
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int I = m.instances;
  // F[i] of this thread: shared [i][lane] or global [i][config]
  double *F = SMEM ? Fs + threadIdx.x : Fg + c;
  const size_t fs = SMEM ? blockDim.x : (size_t)n;
  const kareto_config cf = cfg[c];
  const bool ttl = cf.cap[2] == KARETO_INF;
  const uint64_t Bb = m.block_bytes;
  const kareto_medium md = m.media[cf.medium];
  const double prov_gb = ttl ? m.ttl_prov_gb : (double)(cf.cap[2] * Bb) / 1e9;
  const double bw = qmin(md.bw_max, md.bw_base + md.bw_slope * prov_gb);
  for (int i = 0; i < I; i++) F[i * fs] = 0.0;
  const int64_t a0 = arr[0];
  double total = 0.0;
  uint64_t real = 0, capd = 0;
  for (int64_t r = 0; r < R; r++) {
    const uint4 hc = cnt[(size_t)r * n + c];
    const uint64_t h1 = hc.x, h2 = hc.y, h3 = hc.z;
    const double a = (double)(arr[r] - a0) * 1e-3;  // R50
    int bi = 0;
    double fb = F[0];
    for (int i = 1; i < I; i++) {
      const double f = F[i * fs];
      if (f < fb) { fb = f; bi = i; }
    }
    const double start = qmax(a, fb);
    const double w = start - a;
    const double x = (w * bw) / (double)Bb;  // R51
    const uint64_t h3r = x >= (double)h3 ? h3 : (uint64_t)x;
    const uint64_t H = h1 + h2 + h3r;
    const uint64_t L = inlen[r];
    const uint64_t P0 = m.alpha_ps * L + m.beta_ps * (L * (L - 1) / 2);  // R52
    const uint64_t S = 16 * m.alpha_ps * H + m.beta_ps * (256 * (H * (H - 1) / 2) + 120 * H);
    const double prefill = (double)(P0 - S) * 1e-12;
    const double dram = (double)(h2 * Bb) / m.bw_dram;
    const double decode = (double)(m.dec_ps * (uint64_t)outlen[r]) * 1e-12;
    const double t = (w + prefill) + dram;
    total = total + t;
    if (ttft) ttft[(size_t)c * R + r] = t;
    F[bi * fs] = ((start + prefill) + dram) + decode;
    real += h3r;
    capd += h3;
  }
  double fmax = F[0];
  for (int i = 1; i < I; i++) fmax = qmax(fmax, F[i * fs]);
  const double M = qmax((double)span_ms * 1e-3, fmax);  // R53
  kareto_queue_result q;
  q.ttft_mean_ms = 1e3 * (total / (double)R);
  q.ttft_p99_ms = 0.0;
  q.makespan_s = M;
  q.tokens_per_s = (double)LO / M;
  q.disk_hits_capacity = capd;
  q.disk_hits_realized = real;
  out[c] = q;
}

__global__ void k_pick_p99(const double *__restrict__ sorted, int64_t R, int64_t n, int64_t k,
                           kareto_queue_result *__restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n) out[c].ttft_p99_ms = 1e3 * sorted[(size_t)c * R + (k - 1)];
}

__global__ void k_seg_offsets(int64_t n, int64_t R, int64_t *__restrict__ off) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c <= n) off[c] = c * R;
}

// stack-eligible LRU configurations: per-request counts from the depths (k_queue_counts)
static kareto_status eval_queue_stack(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg, int64_t n,
                                      const uint32_t *ttl_ms, int32_t n_tuner, const kareto_model *model,
                                      kareto_queue_result *out) {
  if (!tr || !model || n < 0 || (n > 0 && (!cfg || !out)) || n_tuner < 0 || (n_tuner > 0 && !ttl_ms))
    return fail(ctx, KARETO_E_INVALID, "eval_queue: bad arguments");
  if (n == 0) return KARETO_OK;
  const int G = tr->K + 1;
  const kareto_model &m = *model;
  if (m.instances < 1 || m.instances > 4096 || m.block_bytes == 0 || !(m.bw_dram > 0) || m.n_media < 1 ||
      m.n_media > 8)
    return fail(ctx, KARETO_E_INVALID, "eval_queue: invalid model constants (1 <= instances <= 4096)");
  std::vector<uint32_t> rows;
  if (n_tuner == 0) rows.assign(G, KARETO_TTL_INF);
  else rows.assign(ttl_ms, ttl_ms + (size_t)n_tuner * G);
  for (int64_t i = 0; i < n; i++) {
    const kareto_config &c = cfg[i];
    if (c.policy != KARETO_LRU) return fail(ctx, KARETO_E_UNSUPPORTED, "eval_queue: config %lld is not LRU", (long long)i);
    if ((n_tuner == 0 && c.tuner != 0) || (n_tuner > 0 && c.tuner >= n_tuner) || c.medium >= m.n_media)
      return fail(ctx, KARETO_E_INVALID, "eval_queue: config %lld: bad tuner / medium", (long long)i);
    const uint32_t *row = rows.data() + (size_t)(n_tuner > 0 ? c.tuner : 0) * G;
    if (c.cap[2] == KARETO_INF) {
      for (int g = 0; g < G; g++)
        if (row[g] == KARETO_TTL_INF) return fail(ctx, KARETO_E_INVALID, "eval_queue: config %lld: TTL mode with an infinite TTL", (long long)i);
    } else {
      for (int g = 1; g < G; g++)
        if (row[g] != row[0])
          return fail(ctx, KARETO_E_UNSUPPORTED, "eval_queue: config %lld: per-group TTLs on a finite disk need the replay",
                      (long long)i);
    }
  }
  cudaStream_t st = ctx->stream;
  const int64_t R = tr->R;
  DBuf<kareto_config> dcfg;
  DBuf<uint32_t> drows;
  DBuf<kareto_queue_result> dout;
  KTRY(dcfg.alloc(ctx, n)); KTRY(drows.alloc(ctx, rows.size())); KTRY(dout.alloc(ctx, n));
  KCUDA(ctx, cudaMemcpyAsync(dcfg.p, cfg, sizeof(kareto_config) * n, cudaMemcpyHostToDevice, st));
  KCUDA(ctx, cudaMemcpyAsync(drows.p, rows.data(), 4 * rows.size(), cudaMemcpyHostToDevice, st));
  // waves sized so the per-configuration TTFT rows (and their sorted copy) fit in free HBM
  double budget = 0;
  KTRY(wave_budget(ctx, 0.4, &budget));
  int64_t W = (int64_t)(budget / (32.0 * (double)R + 8.0 * m.instances + 64.0));
  if (W > n) W = n;
  if (W < 1) return fail(ctx, KARETO_E_OOM, "eval_queue: %lld requests do not fit one configuration", (long long)R);
  const int64_t k99 = (99 * R + 99) / 100;  // ceil(0.99 R)
  const bool smem = (size_t)m.instances * 32 * 8 <= 96 * 1024;
  DBuf<double> F, tt, ts;
  DBuf<uint4> cnt;
  DBuf<int64_t> off;
  DBuf<uint8_t> tmp;
  KTRY(F.alloc(ctx, smem ? 1 : (size_t)m.instances * W)); KTRY(tt.alloc(ctx, (size_t)W * R));
  KTRY(ts.alloc(ctx, (size_t)W * R)); KTRY(cnt.alloc(ctx, (size_t)W * R)); KTRY(off.alloc(ctx, W + 1));
  const size_t sbytes = smem ? (size_t)m.instances * 32 * 8 : 0;
  if (smem) cudaFuncSetAttribute(k_queue<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes);
  KTRY(ensure_depth(ctx, const_cast<kareto_trace *>(tr)));
  for (int64_t w0 = 0; w0 < n; w0 += W) {
    const int64_t nw = n - w0 < W ? n - w0 : W;
    {
      Pass ps(ctx, "F3_counts", 1, 1);
      k_queue_counts<<<(unsigned)(R < 64 * ctx->num_sms ? R : 64 * ctx->num_sms), 128, 0, st>>>(
          tr->s, tr->depth, tr->delta, tr->grp, R, dcfg.p + w0, drows.p, n_tuner, G, nw, cnt.p);
    }
    {
      Pass ps(ctx, "F3_queue", 1, 1);
      const unsigned g = (unsigned)((nw + 31) / 32);
      if (smem)
        k_queue<true><<<g, 32, sbytes, st>>>(tr->arr, tr->inlen, tr->outlen, R, dcfg.p + w0, nw, cnt.p, m,
                                             (uint64_t)tr->span_ms, tr->Ltok + tr->O, F.p, tt.p, dout.p + w0);
      else
        k_queue<false><<<g, 32, 0, st>>>(tr->arr, tr->inlen, tr->outlen, R, dcfg.p + w0, nw, cnt.p, m,
                                         (uint64_t)tr->span_ms, tr->Ltok + tr->O, F.p, tt.p, dout.p + w0);
    }
    {
      Pass ps(ctx, "F3_p99", 1, 2);
      k_seg_offsets<<<grid_for(nw + 1, 256), 256, 0, st>>>(nw, R, off.p);
      size_t bytes = 0;
      KCUDA(ctx, cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, tt.p, ts.p, nw * R, nw, off.p, off.p + 1, st));
      if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
      bytes = tmp.n;
      KCUDA(ctx, cub::DeviceSegmentedSort::SortKeys(tmp.p, bytes, tt.p, ts.p, nw * R, nw, off.p, off.p + 1, st));
      k_pick_p99<<<grid_for(nw, 256), 256, 0, st>>>(ts.p, R, nw, k99, dout.p + w0);
    }
  }
  KCUDA(ctx, cudaMemcpyAsync(out, dout.p, sizeof(kareto_queue_result) * n, cudaMemcpyDeviceToHost, st));
  return sync(ctx, "eval_queue");
}

// all configurations: stack-eligible LRU ones through the depth counts, the others through the
// K6 replay with the queue evaluated inline (the hit prefix of every request, R49)
static kareto_status eval_queue(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg, int64_t n,
                                const uint32_t *ttl_ms, int32_t n_tuner, const kareto_model *model,
                                kareto_queue_result *out) {
  if (!tr || !model || n < 0 || (n > 0 && (!cfg || !out)) || n_tuner < 0 || (n_tuner > 0 && !ttl_ms))
    return fail(ctx, KARETO_E_INVALID, "eval_queue: bad arguments");
  if (n == 0) return KARETO_OK;
  const int G = tr->K + 1;
  const kareto_model &m = *model;
  if (m.instances < 1 || m.instances > 4096 || m.block_bytes == 0 || !(m.bw_dram > 0) || m.n_media < 1 ||
      m.n_media > 8)
    return fail(ctx, KARETO_E_INVALID, "eval_queue: invalid model constants (1 <= instances <= 4096)");
  std::vector<uint32_t> rows;
  if (n_tuner == 0) rows.assign(G, KARETO_TTL_INF);
  else rows.assign(ttl_ms, ttl_ms + (size_t)n_tuner * G);
  std::vector<kareto_config> cS, cP;
  std::vector<int64_t> iS, iP;
  for (int64_t i = 0; i < n; i++) {
    const kareto_config &c = cfg[i];
    if (c.policy > KARETO_LFU) return fail(ctx, KARETO_E_INVALID, "eval_queue: config %lld: bad policy", (long long)i);
    if ((n_tuner == 0 && c.tuner != 0) || (n_tuner > 0 && c.tuner >= n_tuner) || c.medium >= m.n_media)
      return fail(ctx, KARETO_E_INVALID, "eval_queue: config %lld: bad tuner / medium", (long long)i);
    const uint32_t *row = rows.data() + (size_t)(n_tuner > 0 ? c.tuner : 0) * G;
    bool uniform = true;
    for (int g = 1; g < G; g++) uniform = uniform && row[g] == row[0];
    if (c.cap[2] == KARETO_INF) {
      for (int g = 0; g < G; g++)
        if (row[g] == KARETO_TTL_INF)
          return fail(ctx, KARETO_E_INVALID, "eval_queue: config %lld: TTL mode with an infinite TTL", (long long)i);
    }
    const bool stack = c.policy == KARETO_LRU && (c.cap[2] == KARETO_INF || uniform);
    (stack ? cS : cP).push_back(c);
    (stack ? iS : iP).push_back(i);
  }
  std::vector<kareto_queue_result> oS(cS.size()), oP(cP.size());
  if (!cS.empty())
    KTRY(eval_queue_stack(ctx, tr, cS.data(), (int64_t)cS.size(), ttl_ms, n_tuner, model, oS.data()));
  if (!cP.empty()) {
    DBuf<uint32_t> drows;
    DBuf<kareto_counts> dcnt;
    DBuf<kareto_queue_result> dq;
    KTRY(drows.alloc(ctx, rows.size())); KTRY(dcnt.alloc(ctx, cP.size())); KTRY(dq.alloc(ctx, cP.size()));
    KCUDA(ctx, cudaMemcpyAsync(drows.p, rows.data(), 4 * rows.size(), cudaMemcpyHostToDevice, ctx->stream));
    QueueArgs qa;
    qa.model = model;
    qa.out_dev = dq.p;
    qa.span_ms = (uint64_t)tr->span_ms;
    qa.LO = tr->Ltok + tr->O;
    KTRY(replay_eval(ctx, const_cast<kareto_trace *>(tr), cP.data(), (int64_t)cP.size(), rows.data(), drows.p,
                     n_tuner, dcnt.p, qa));
    KCUDA(ctx, cudaMemcpyAsync(oP.data(), dq.p, sizeof(kareto_queue_result) * cP.size(), cudaMemcpyDeviceToHost,
                               ctx->stream));
    KTRY(sync(ctx, "eval_queue replay"));
  }
  for (size_t k = 0; k < cS.size(); k++) out[iS[k]] = oS[k];
  for (size_t k = 0; k < cP.size(); k++) out[iP[k]] = oP[k];
  return KARETO_OK;
}

}  // namespace kareto

extern "C" kareto_status kareto_eval_queue(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg,
                                           int64_t n_cfg, const uint32_t *ttl_ms, int32_t n_tuner,
                                           const kareto_model *model, kareto_queue_result *out) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->err.clear();
  if (tr && tr->sharded)
    return kareto::fail(ctx, KARETO_E_UNSUPPORTED, "%s needs the whole trace (not a time shard)", "kareto_eval_queue");
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::eval_queue(ctx, tr, cfg, n_cfg, ttl_ms, n_tuner, model, out);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

// replay.cu -- row a7, K6: literal per-configuration tier replay for the configurations the
// stack path cannot cover (FIFO, LFU, and LRU with per-group disk TTLs on a finite disk).
//
// Semantics = DESIGN.md "Replay semantics" (R9-R24): per request, purge
// expired disk blocks (CAPACITY mode), look up the longest present prefix on the
// pre-request state, then touch the chain leaf -> root, each touch promoting to HBM and
// cascading policy victims one tier down (TTL mode: HBM -> DRAM -> drop, with a
// write-through lease store billed by C_g).
//
// Layout (B200): one thread per configuration; a wave of W configurations walks the same
// access stream in lockstep, and every per-(block, configuration) field is stored at
// [block * W + config], so the 32 lanes of a warp touching the same block hit one or two
// sectors.  Victim order: LRU / FIFO tiers are doubly-linked lists (front = newest key;
// for LRU a demoted block's last_seq exceeds every member of the lower tier, so demotion
// order is key order), LFU tiers are binary heaps keyed (freq, last_seq); disk purges use a
// binary heap keyed last_t + tau_g.  All state lives in HBM; waves are sized to free memory.
#include "replay.cuh"

namespace kareto {

enum : uint8_t { T_NONE = 0, T_HBM = 1, T_DRAM = 2, T_DISK = 3 };

struct RView {
  uint8_t *tier;
  uint32_t *lp, *ln, *lseq, *iseq, *freq, *last_t, *lease, *epos;
  uint32_t *heap[3];  // LFU heaps per tier, [slot * W + c]
  uint32_t *eheap;    // expiry heap
  const uint16_t *gblk;
  uint64_t W;
  uint32_t c;
  __device__ __forceinline__ uint64_t at(uint32_t b) const { return (uint64_t)b * W + c; }
};

struct RCfg {
  uint64_t cap[3];
  int policy;
  bool ttl_mode, use_expiry;
  const uint32_t *tau;  // [G]
  uint32_t head[3], tail[3];
  uint64_t size[3];
  uint32_t esize;
  uint32_t seq;
  kareto_counts k;
};

// ---------------------------------------------------------------- lists (LRU / FIFO)
__device__ __forceinline__ void l_push_front(const RView &v, RCfg &s, int t, uint32_t b) {
  uint32_t h = s.head[t - 1];
  v.ln[v.at(b)] = h;
  v.lp[v.at(b)] = kNone;
  if (h != kNone) v.lp[v.at(h)] = b; else s.tail[t - 1] = b;
  s.head[t - 1] = b;
}
__device__ __forceinline__ void l_unlink(const RView &v, RCfg &s, int t, uint32_t b) {
  uint32_t p = v.lp[v.at(b)], n = v.ln[v.at(b)];
  if (p != kNone) v.ln[v.at(p)] = n; else s.head[t - 1] = n;
  if (n != kNone) v.lp[v.at(n)] = p; else s.tail[t - 1] = p;
}

// ---------------------------------------------------------------- heaps (LFU, expiry)
__device__ __forceinline__ uint64_t lfu_key(const RView &v, uint32_t b) {
  return ((uint64_t)v.freq[v.at(b)] << 32) | v.lseq[v.at(b)];
}
// position of b in its tier heap is kept in lp[] for LFU
__device__ void h_swap(const RView &v, uint32_t *hp, uint64_t i, uint64_t j) {
  uint32_t a = hp[i * v.W + v.c], b = hp[j * v.W + v.c];
  hp[i * v.W + v.c] = b;
  hp[j * v.W + v.c] = a;
  v.lp[v.at(b)] = (uint32_t)i;
  v.lp[v.at(a)] = (uint32_t)j;
}
__device__ void h_up(const RView &v, uint32_t *hp, uint64_t i) {
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (lfu_key(v, hp[i * v.W + v.c]) >= lfu_key(v, hp[p * v.W + v.c])) break;
    h_swap(v, hp, i, p);
    i = p;
  }
}
__device__ void h_down(const RView &v, uint32_t *hp, uint64_t n, uint64_t i) {
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && lfu_key(v, hp[l * v.W + v.c]) < lfu_key(v, hp[m * v.W + v.c])) m = l;
    if (r < n && lfu_key(v, hp[r * v.W + v.c]) < lfu_key(v, hp[m * v.W + v.c])) m = r;
    if (m == i) break;
    h_swap(v, hp, i, m);
    i = m;
  }
}

__device__ __forceinline__ uint64_t exp_key(const RView &v, const RCfg &s, uint32_t b) {
  return (uint64_t)v.last_t[v.at(b)] + s.tau[v.gblk[b]];
}
__device__ void e_swap(const RView &v, uint64_t i, uint64_t j) {
  uint32_t a = v.eheap[i * v.W + v.c], b = v.eheap[j * v.W + v.c];
  v.eheap[i * v.W + v.c] = b;
  v.eheap[j * v.W + v.c] = a;
  v.epos[v.at(b)] = (uint32_t)i;
  v.epos[v.at(a)] = (uint32_t)j;
}
__device__ void e_up(const RView &v, const RCfg &s, uint64_t i) {
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (exp_key(v, s, v.eheap[i * v.W + v.c]) >= exp_key(v, s, v.eheap[p * v.W + v.c])) break;
    e_swap(v, i, p);
    i = p;
  }
}
__device__ void e_down(const RView &v, const RCfg &s, uint64_t i) {
  uint64_t n = s.esize;
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && exp_key(v, s, v.eheap[l * v.W + v.c]) < exp_key(v, s, v.eheap[m * v.W + v.c])) m = l;
    if (r < n && exp_key(v, s, v.eheap[r * v.W + v.c]) < exp_key(v, s, v.eheap[m * v.W + v.c])) m = r;
    if (m == i) break;
    e_swap(v, i, m);
    i = m;
  }
}
__device__ void e_push(const RView &v, RCfg &s, uint32_t b) {
  uint64_t i = s.esize++;
  v.eheap[i * v.W + v.c] = b;
  v.epos[v.at(b)] = (uint32_t)i;
  e_up(v, s, i);
}
__device__ void e_remove(const RView &v, RCfg &s, uint32_t b) {
  uint64_t i = v.epos[v.at(b)], last = --s.esize;
  if (i != last) {
    e_swap(v, i, last);
    e_up(v, s, i);
    e_down(v, s, i);
  }
  v.epos[v.at(b)] = kNone;
}

// ---------------------------------------------------------------- tier operations
__device__ void t_insert(const RView &v, RCfg &s, int t, uint32_t b) {
  v.tier[v.at(b)] = (uint8_t)t;
  if (s.policy == KARETO_LFU) {
    uint32_t *hp = v.heap[t - 1];
    uint64_t i = s.size[t - 1];
    hp[i * v.W + v.c] = b;
    v.lp[v.at(b)] = (uint32_t)i;
    s.size[t - 1]++;
    h_up(v, hp, i);
  } else {
    l_push_front(v, s, t, b);
    s.size[t - 1]++;
  }
  if (t == T_DISK && s.use_expiry && s.tau[v.gblk[b]] != KARETO_TTL_INF) e_push(v, s, b);
}
__device__ void t_remove(const RView &v, RCfg &s, int t, uint32_t b) {
  if (s.policy == KARETO_LFU) {
    uint32_t *hp = v.heap[t - 1];
    uint64_t i = v.lp[v.at(b)], last = --s.size[t - 1];
    if (i != last) {
      h_swap(v, hp, i, last);
      h_up(v, hp, i);
      h_down(v, hp, s.size[t - 1], i);
    }
  } else {
    l_unlink(v, s, t, b);
    s.size[t - 1]--;
  }
  if (t == T_DISK && v.epos[v.at(b)] != kNone) e_remove(v, s, b);
}
__device__ __forceinline__ uint32_t t_victim(const RView &v, const RCfg &s, int t) {
  return s.policy == KARETO_LFU ? v.heap[t - 1][v.c] : s.tail[t - 1];
}
// reorder after an HBM hit (LRU: move to front; LFU: key grew)
__device__ void t_touch_hbm(const RView &v, RCfg &s, uint32_t b) {
  if (s.policy == KARETO_LRU) {
    l_unlink(v, s, T_HBM, b);
    l_push_front(v, s, T_HBM, b);
  } else if (s.policy == KARETO_LFU) {
    h_down(v, v.heap[0], s.size[0], v.lp[v.at(b)]);
  }
}

// CASCADE from HBM after an insertion: each level overflows by at most one block
__device__ void cascade(const RView &v, RCfg &s) {
  for (int t = T_HBM; t <= T_DISK; t++) {
    uint64_t capt = (t == T_DISK && s.ttl_mode) ? 0 : s.cap[t - 1];
    if (s.size[t - 1] <= capt) return;
    uint32_t x = t_victim(v, s, t);
    t_remove(v, s, t, x);
    s.k.evict[t - 1] += 1;
    bool next = s.ttl_mode ? (t == T_HBM) : (t < T_DISK);
    if (!next) {
      v.tier[v.at(x)] = T_NONE;
      return;
    }
    s.seq += 1;
    v.iseq[v.at(x)] = s.seq;  // last_seq kept (FIFO order of the lower tier = entry order)
    t_insert(v, s, t + 1, x);
  }
}

__global__ void __launch_bounds__(128) k_replay(ReplayTrace T, const kareto_config *__restrict__ cfg,
                                                const uint32_t *__restrict__ rows, int n_tuner, int G, RView v0,
                                                int64_t n, kareto_counts *__restrict__ out) {
  const int64_t ci = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ci >= n) return;
  RView v = v0;
  v.c = (uint32_t)ci;
  RCfg s;
  const kareto_config c = cfg[ci];
  s.cap[0] = c.cap[0];
  s.cap[1] = c.cap[1];
  s.cap[2] = c.cap[2];
  s.policy = c.policy;
  s.ttl_mode = c.cap[2] == KARETO_INF;
  s.tau = rows + (size_t)(n_tuner > 0 ? c.tuner : 0) * G;
  bool any_finite = false;
  for (int g = 0; g < G; g++) any_finite |= s.tau[g] != KARETO_TTL_INF;
  s.use_expiry = !s.ttl_mode && any_finite;
  for (int t = 0; t < 3; t++) { s.head[t] = s.tail[t] = kNone; s.size[t] = 0; }
  s.esize = 0;
  s.seq = 0;
  memset(&s.k, 0, sizeof(s.k));
  for (uint32_t r = 0; r < T.R; r++) {
    const uint32_t s0 = T.s[r], nb = T.s[r + 1] - s0;
    if (nb == 0) continue;
    const uint32_t a = T.arr[r];
    const uint32_t tg = s.tau[T.grp[r]];
    // 1 PURGE (CAPACITY mode): disk blocks with a - last_t > tau_g
    if (s.use_expiry) {
      while (s.esize > 0) {
        uint32_t x = v.eheap[v.c];
        if (exp_key(v, s, x) >= a) break;
        t_remove(v, s, T_DISK, x);  // also leaves the expiry heap
        v.tier[v.at(x)] = T_NONE;
      }
    }
    // 2 LOOKUP on the pre-request state (block k sits at position s0 + nb - 1 - k)
    bool in_prefix = true;
    for (uint32_t k = 0; k < nb; k++) {
      const uint32_t b = T.blk[s0 + nb - 1 - k];
      const uint8_t t = v.tier[v.at(b)];
      const uint32_t ls = v.lease[v.at(b)];  // kNone = never seen
      const bool alive = ls != kNone && (a - ls) <= tg;
      const bool present = t != T_NONE || (s.ttl_mode && alive);
      if (in_prefix && !present) in_prefix = false;
      if (in_prefix) {
        s.k.hit[(t != T_NONE ? t : T_DISK) - 1] += 1;
        s.k.hit_pos_sum += k;
      } else {
        s.k.miss += 1;
        if (t != T_NONE) s.k.resident_after_hole += 1;
      }
      if (s.ttl_mode && !alive) s.k.disk_writes += 1;
    }
    // 3 UPDATE leaf -> root
    for (uint32_t kk = nb; kk-- > 0;) {
      const uint32_t b = T.blk[s0 + nb - 1 - kk];
      s.seq += 1;
      const uint8_t t = v.tier[v.at(b)];
      if (t == T_HBM) {
        if (s.policy == KARETO_LRU) { v.lseq[v.at(b)] = s.seq; t_touch_hbm(v, s, b); }
        else if (s.policy == KARETO_LFU) { v.freq[v.at(b)] += 1; v.lseq[v.at(b)] = s.seq; t_touch_hbm(v, s, b); }
      } else {
        if (t == T_DRAM || t == T_DISK) {
          t_remove(v, s, t, b);
          v.freq[v.at(b)] += 1;  // LFU count carried across tiers
        } else {
          v.freq[v.at(b)] = 1;
        }
        v.lseq[v.at(b)] = s.seq;
        v.iseq[v.at(b)] = s.seq;
        t_insert(v, s, T_HBM, b);
        cascade(v, s);
      }
      const uint32_t ls = v.lease[v.at(b)];
      if (s.ttl_mode && ls != kNone) {
        uint32_t dt = a - ls;
        s.k.bytetime_block_ms += dt < tg ? dt : tg;
      }
      v.last_t[v.at(b)] = a;
      if (v.tier[v.at(b)] == T_DISK && v.epos[v.at(b)] != kNone) {  // demoted in its own cascade
        e_up(v, s, v.epos[v.at(b)]);
        e_down(v, s, v.epos[v.at(b)]);
      }
      v.lease[v.at(b)] = a;
    }
  }
  if (s.ttl_mode) {
    for (uint32_t b = 0; b < T.U; b++)
      if (v.lease[v.at(b)] != kNone) s.k.bytetime_block_ms += s.tau[v.gblk[b]];
    s.k.evict[2] = 0;
  } else {
    s.k.disk_writes = s.cap[2] > 0 ? s.k.evict[1] : 0;
    if (any_finite) s.k.evict[2] = KARETO_NA;
  }
  out[ci] = s.k;
}

// ---------------------------------------------------------------- dense block ids
__global__ void k_first_init(uint64_t N, const uint32_t *__restrict__ prev, uint32_t *__restrict__ f,
                             uint32_t *__restrict__ isfirst) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t p = prev[j];
    f[j] = p == kNone ? (uint32_t)j : p;
    isfirst[j] = p == kNone;
  }
}
__global__ void k_first_jump(uint64_t N, const uint32_t *__restrict__ fin, uint32_t *__restrict__ fout,
                             int *__restrict__ changed) {
  int ch = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a = fin[j], b = fin[a];
    fout[j] = b;
    ch |= (a != b);
  }
  if (__syncthreads_or(ch) && threadIdx.x == 0) atomicOr(changed, 1);
}
__global__ void k_dense_ids(uint64_t N, const uint32_t *__restrict__ f, const uint32_t *__restrict__ idfirst,
                            const uint32_t *__restrict__ prev, const uint32_t *__restrict__ req,
                            const uint16_t *__restrict__ grp, uint32_t *__restrict__ blk, uint16_t *__restrict__ gblk) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t id = idfirst[f[j]];
    blk[j] = id;
    if (prev[j] == kNone) gblk[id] = grp[req[j]];
  }
}
__global__ void k_arr_rel(int64_t R, const int64_t *__restrict__ arr, uint32_t *__restrict__ rel) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
    rel[r] = (uint32_t)(arr[r] - arr[0]);
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

kareto_status replay_prepare(kareto_ctx *ctx, kareto_trace *tr) {
  if (tr->blk || tr->N == 0) return KARETO_OK;
  if (tr->span_ms >= (int64_t)kNone - 1) return fail(ctx, KARETO_E_OVERFLOW, "trace span >= 2^32-1 ms");
  cudaStream_t st = ctx->stream;
  const uint64_t N = (uint64_t)tr->N;
  const int sms = ctx->num_sms;
  DBuf<uint32_t> f0, f1, isf, idf;
  DBuf<int> changed;
  DBuf<uint8_t> tmp;
  KTRY(f0.alloc(ctx, N)); KTRY(f1.alloc(ctx, N)); KTRY(isf.alloc(ctx, N)); KTRY(idf.alloc(ctx, N));
  KTRY(changed.alloc(ctx, 1));
  Pass ps(ctx, "K6_dense_ids", 1, 3);
  k_first_init<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->prev, f0.p, isf.p);
  for (int it = 0; it < 40; it++) {  // pointer jumping to the first occurrence
    KTRY(changed.zero());
    k_first_jump<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, f0.p, f1.p, changed.p);
    ctx->own_launches++;
    std::swap(f0.p, f1.p);
    int h = 0;
    KCUDA(ctx, cudaMemcpyAsync(&h, changed.p, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    if (!h) break;
  }
  KTRY(cub_tmp(ctx, tmp, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, isf.p, idf.p, (int64_t)N, st);
  }));
  KCUDA(ctx, cudaMallocAsync((void **)&tr->blk, 4 * N, st));
  KCUDA(ctx, cudaMallocAsync((void **)&tr->gblk, 2 * (size_t)(tr->U > 0 ? tr->U : 1), st));
  KCUDA(ctx, cudaMallocAsync((void **)&tr->arr_rel, 4 * (size_t)tr->R, st));
  k_dense_ids<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, f0.p, idf.p, tr->prev, tr->req, tr->grp, tr->blk, tr->gblk);
  k_arr_rel<<<grid_for(tr->R, 256, 4 * sms), 256, 0, st>>>(tr->R, tr->arr, tr->arr_rel);
  return KARETO_OK;
}

kareto_status replay_eval(kareto_ctx *ctx, kareto_trace *tr, const kareto_config *cfg_host, int64_t n,
                          const uint32_t *rows_dev, int n_tuner, kareto_counts *counts_dev) {
  if (n <= 0) return KARETO_OK;
  KTRY(replay_prepare(ctx, tr));
  cudaStream_t st = ctx->stream;
  const uint64_t U = tr->U > 0 ? (uint64_t)tr->U : 1;
  ReplayTrace T{(uint32_t)tr->R, (uint32_t)tr->U, tr->s, tr->arr_rel, tr->grp, tr->blk};
  // wave size from free memory: per (block, config) 1 + 8*4 bytes + heaps 4*4 bytes
  size_t freeb = 0, totb = 0;
  KCUDA(ctx, cudaMemGetInfo(&freeb, &totb));
  const uint64_t per_cfg = U * (1 + 8 * 4 + 4 * 4) + 64;
  uint64_t W = (uint64_t)(0.5 * (double)freeb) / per_cfg;
  if (W > 16384) W = 16384;
  if (W > (uint64_t)n) W = (uint64_t)n;
  if (W < 1) return fail(ctx, KARETO_E_OOM, "replay needs %llu bytes per configuration", (unsigned long long)per_cfg);
  DBuf<uint8_t> tier;
  DBuf<uint32_t> lp, ln, lseq, iseq, freq, last_t, lease, epos, heap, eheap;
  KTRY(tier.alloc(ctx, U * W));
  for (DBuf<uint32_t> *b : {&lp, &ln, &lseq, &iseq, &freq, &last_t, &lease, &epos, &eheap}) KTRY(b->alloc(ctx, U * W));
  KTRY(heap.alloc(ctx, 3 * (U + 2) * W));
  DBuf<kareto_config> dcfg;
  KTRY(dcfg.alloc(ctx, n));
  KCUDA(ctx, cudaMemcpyAsync(dcfg.p, cfg_host, sizeof(kareto_config) * n, cudaMemcpyHostToDevice, st));
  for (int64_t w0 = 0; w0 < n; w0 += (int64_t)W) {
    int64_t nw = n - w0 < (int64_t)W ? n - w0 : (int64_t)W;
    KCUDA(ctx, cudaMemsetAsync(tier.p, 0, U * W, st));
    KCUDA(ctx, cudaMemsetAsync(lease.p, 0xFF, 4 * U * W, st));
    KCUDA(ctx, cudaMemsetAsync(epos.p, 0xFF, 4 * U * W, st));
    KCUDA(ctx, cudaMemsetAsync(freq.p, 0, 4 * U * W, st));
    RView v{};
    v.tier = tier.p; v.lp = lp.p; v.ln = ln.p; v.lseq = lseq.p; v.iseq = iseq.p; v.freq = freq.p;
    v.last_t = last_t.p; v.lease = lease.p; v.epos = epos.p;
    v.heap[0] = heap.p; v.heap[1] = heap.p + (U + 2) * W; v.heap[2] = heap.p + 2 * (U + 2) * W;
    v.eheap = eheap.p;
    v.gblk = tr->gblk;
    v.W = W;
    Pass ps(ctx, "K6_replay", 1, 1);
    k_replay<<<grid_for(nw, 128), 128, 0, st>>>(T, dcfg.p + w0, rows_dev, n_tuner, tr->K + 1, v, nw, counts_dev + w0);
  }
  return sync(ctx, "replay");
}

}  // namespace kareto

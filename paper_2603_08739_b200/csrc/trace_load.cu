// trace_load.cu -- kareto_load_trace: rows a1 (ingest), a2 (K1 chained block hash) and
// a3 (K2 previous access / reuse interval / chain check / prefix-subtree groups) of the
// hot path; a4 (K3 LRU depth) lives in stack_depth.cu.
//
//   a1  requests stable-sorted by (arrival, file index) (R6); blocks are
//       the full 16-token blocks of each input (R1, R3); touch order: request by
//       request, blocks leaf -> root (R12), so request r owns positions [s_r, s_r + n_r)
//       and block k sits at s_r + n_r - 1 - k.
//   a2  K1 chain hash (R2): c_k = fmix64(NH(t[16k..16k+15])), P_k = R P_{k-1} + c_k,
//       h_k = fmix64(P_k) -- an affine recurrence, computed as a segmented parallel
//       scan instead of a serial per-request chain.
//   a3  K2: radix sort (hash, position) [CUB], link equal neighbours -> prev, then one
//       coalesced pass for delta (P:748-756 inter-arrival times), the chain check (R7),
//       and per-request first/reuse counts; groups = top-K prefix subtrees by reuse
//       (R23).
#include <cub/cub.cuh>

#include "trace_load.cuh"
#include "bucket_link.cuh"

namespace kareto {

template <typename F>
static kareto_status cub_call(kareto_ctx *ctx, DBuf<uint8_t> &tmp, F &&f) {
  size_t bytes = 0;
  KCUDA(ctx, f((void *)nullptr, bytes));
  if (bytes > tmp.n) KTRY(tmp.alloc(ctx, bytes));
  size_t b2 = tmp.n;
  KCUDA(ctx, f((void *)tmp.p, b2));
  return KARETO_OK;
}

// ------------------------------------------------------------------ a1 ----
// order-preserving signed -> unsigned key, and its min / max (the sort then covers only the bits
// of max - min: a 2-hour trace needs ~23 bits, i.e. 3 radix passes instead of 8)
__global__ void k_sort_keys(const int64_t *__restrict__ arrival, int64_t R, uint64_t *__restrict__ key,
                            uint32_t *__restrict__ idx, unsigned long long *__restrict__ mnmx) {
  unsigned long long mn = ~0ull, mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = (uint64_t)arrival[i] ^ 0x8000000000000000ULL;
    key[i] = k;
    idx[i] = (uint32_t)i;
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mnmx[0], mn);
    atomicMax(&mnmx[1], mx);
  }
}
__global__ void k_rebase_keys(uint64_t *__restrict__ key, int64_t R, const unsigned long long *__restrict__ mnmx) {
  const uint64_t mn = mnmx[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x)
    key[i] -= mn;
}

__global__ void k_req_meta(int64_t R, int mode, const uint32_t *__restrict__ order, const int64_t *__restrict__ arrival,
                           const int32_t *__restrict__ out_tok, const int64_t *__restrict__ offsets,
                           const int64_t *__restrict__ input_tokens, int64_t *__restrict__ arr_sorted,
                           int64_t *__restrict__ src_off, uint64_t *__restrict__ nblk, uint32_t *__restrict__ inlen,
                           uint32_t *__restrict__ outlen, LoadStats *st) {
  unsigned long long sl_lo = 0, sl_hi = 0, sq_lo = 0, sq_hi = 0, O = 0;
  unsigned int flags = 0, maxb = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t f = order[r];
    int64_t a = arrival[f];
    arr_sorted[r] = a;
    int64_t o0 = offsets[f], o1 = offsets[f + 1];
    int64_t cnt = o1 - o0;
    if (cnt < 0) { flags |= F_OFFSETS; cnt = 0; }
    int32_t ot = out_tok[f];
    if (ot < 0) { flags |= F_OUTPUT; ot = 0; }
    O += (unsigned long long)ot;
    uint64_t n, L;
    if (mode == KARETO_TOKENS) {
      L = (uint64_t)cnt;
      n = L / 16;
    } else {
      n = (uint64_t)cnt;
      int64_t li = input_tokens ? input_tokens[f] : (int64_t)(16 * n);
      if (li < (int64_t)(16 * n)) { flags |= F_INPUT_LEN; li = (int64_t)(16 * n); }
      L = (uint64_t)li;
    }
    src_off[r] = o0;
    nblk[r] = n;
    if (L > 0xFFFFFFFFull) flags |= F_INPUT_LEN;
    inlen[r] = L > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)L;
    outlen[r] = (uint32_t)ot;
    if (n > maxb) maxb = n > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)n;
    // exact 128-bit sums split into 32-bit halves: SL = sum L, SQ = sum L(L-1)/2
    unsigned __int128 q = L ? ((unsigned __int128)L * (unsigned __int128)(L - 1)) / 2 : 0;
    sl_lo += L & 0xFFFFFFFFull;
    sl_hi += L >> 32;
    uint64_t q64 = (uint64_t)q;  // L < 2^32 in any sane trace; the high part is flagged below
    if ((q >> 64) != 0) flags |= F_INPUT_LEN;
    sq_lo += q64 & 0xFFFFFFFFull;
    sq_hi += q64 >> 32;
  }
  // warp-level reduction, one atomic per warp
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sl_lo += __shfl_xor_sync(0xffffffffu, sl_lo, off);
    sl_hi += __shfl_xor_sync(0xffffffffu, sl_hi, off);
    sq_lo += __shfl_xor_sync(0xffffffffu, sq_lo, off);
    sq_hi += __shfl_xor_sync(0xffffffffu, sq_hi, off);
    O += __shfl_xor_sync(0xffffffffu, O, off);
    flags |= __shfl_xor_sync(0xffffffffu, flags, off);
    unsigned mb = __shfl_xor_sync(0xffffffffu, maxb, off);
    maxb = mb > maxb ? mb : maxb;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&st->sl_lo, sl_lo);
    atomicAdd(&st->sl_hi, sl_hi);
    atomicAdd(&st->sq_lo, sq_lo);
    atomicAdd(&st->sq_hi, sq_hi);
    atomicAdd(&st->O, O);
    if (flags) atomicOr(&st->flags, flags);
    atomicMax(&st->max_blocks, maxb);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->arr_first = arr_sorted[0];
  }
}

__global__ void k_narrow_starts(int64_t R, const uint64_t *__restrict__ s64, uint32_t *__restrict__ s32,
                                const int64_t *__restrict__ arr_sorted, LoadStats *st) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= R; r += (int64_t)gridDim.x * blockDim.x)
    s32[r] = (uint32_t)s64[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->n_total = s64[R];
    st->arr_first = arr_sorted[0];
    st->arr_last = arr_sorted[R - 1];
  }
}

// ------------------------------------------------------------------ a2: K1 ----
// Segmented scan element: x -> a*x + b.  combine(earlier e, later l) = (l.a*e.a, l.a*e.b + l.b)
struct Aff {
  uint64_t a, b;
};
__device__ __forceinline__ Aff aff_compose(Aff e, Aff l) { return {l.a * e.a, l.a * e.b + l.b}; }

__device__ __forceinline__ uint64_t nh_block(const uint32_t t[16], const uint32_t key[16]) {
  uint64_t acc = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    uint32_t a = t[2 * j] + key[2 * j];
    uint32_t b = t[2 * j + 1] + key[2 * j + 1];
    acc += (uint64_t)a * (uint64_t)b;
    acc += ((uint64_t)t[2 * j + 1] << 32) | (uint64_t)t[2 * j];
  }
  return fmix64(acc);
}

// Load the 16 tokens of a block starting at word pointer p (4-byte aligned).  Vector
// loads of the covering 16-byte chunks + a two-level funnel select; a scalar fallback
// near the end of the token buffer avoids reading past it.
__device__ __forceinline__ void load_block_tokens(const uint32_t *p, const uint32_t *end, uint32_t t[16]) {
  uintptr_t addr = (uintptr_t)p;
  int mis = (int)((addr >> 2) & 3);
  const uint4 *q = (const uint4 *)(addr & ~(uintptr_t)15);
  if (mis != 0 && (const uint32_t *)(q + 5) > end) {
#pragma unroll
    for (int i = 0; i < 16; i++) t[i] = __ldg(p + i);
    return;
  }
  uint32_t w[20];
  uint4 c0 = __ldg(q), c1 = __ldg(q + 1), c2 = __ldg(q + 2), c3 = __ldg(q + 3);
  uint4 c4 = mis ? __ldg(q + 4) : make_uint4(0, 0, 0, 0);
  w[0] = c0.x; w[1] = c0.y; w[2] = c0.z; w[3] = c0.w;
  w[4] = c1.x; w[5] = c1.y; w[6] = c1.z; w[7] = c1.w;
  w[8] = c2.x; w[9] = c2.y; w[10] = c2.z; w[11] = c2.w;
  w[12] = c3.x; w[13] = c3.y; w[14] = c3.z; w[15] = c3.w;
  w[16] = c4.x; w[17] = c4.y; w[18] = c4.z; w[19] = c4.w;
  uint32_t u[18];
#pragma unroll
  for (int i = 0; i < 18; i++) u[i] = (mis & 1) ? w[i + 1] : w[i];
#pragma unroll
  for (int i = 0; i < 16; i++) t[i] = (mis & 2) ? u[i + 2] : u[i];
}

// Half a block (8 tokens) starting at word pointer p: the 2 or 3 covering 16-byte chunks
// + funnel select.  Two threads per block halve the lines one warp-wide load touches
// (adjacent lanes read adjacent 32 B), i.e. the L1 wavefronts per block.
__device__ __forceinline__ void load_half_tokens(const uint32_t *p, const uint32_t *end, uint32_t t[8]) {
  uintptr_t addr = (uintptr_t)p;
  int mis = (int)((addr >> 2) & 3);
  const uint4 *q = (const uint4 *)(addr & ~(uintptr_t)15);
  if ((const uint32_t *)(q + (mis ? 3 : 2)) > end) {
#pragma unroll
    for (int i = 0; i < 8; i++) t[i] = __ldg(p + i);
    return;
  }
  uint32_t w[12];
  uint4 c0 = __ldg(q), c1 = __ldg(q + 1);
  uint4 c2 = mis ? __ldg(q + 2) : make_uint4(0, 0, 0, 0);
  w[0] = c0.x; w[1] = c0.y; w[2] = c0.z; w[3] = c0.w;
  w[4] = c1.x; w[5] = c1.y; w[6] = c1.z; w[7] = c1.w;
  w[8] = c2.x; w[9] = c2.y; w[10] = c2.z; w[11] = c2.w;
  uint32_t u[10];
#pragma unroll
  for (int i = 0; i < 10; i++) u[i] = (mis & 1) ? w[i + 1] : w[i];
#pragma unroll
  for (int i = 0; i < 8; i++) t[i] = (mis & 2) ? u[i + 2] : u[i];
}

// 2 warps per CTA: a warp whose request-aligned range holds a long request (agent contexts up to
// 8K blocks) keeps only its partner idle, not 7 (config 4: 1.83 -> 1.75 ms; 32 resident CTAs of
// 64 threads still fill an SM)
constexpr int K1_THREADS = 64;
constexpr int K1_WARPS = K1_THREADS / 32;

// Every WARP owns a request-aligned range of sorted blocks [s[rb], s[re)) (rb, re = first
// requests starting at or after w*N/nWarps and (w+1)*N/nWarps), so the scan carry never
// crosses warps: rounds of 32 consecutive blocks, one thread per block, a 5-step shuffle
// scan and the carry kept in a register -- no block-level barrier on the path, so the
// warps of an SM overlap each other's load latency freely.
//
// Time-sharded loads hash only the requests [r0, r1): s, tok_off point at request r0, positions
// are global (pos_base = s[0]), outputs are indexed by position - pos_base, and req_out holds
// global request indices (r + req_base).
__global__ void __launch_bounds__(K1_THREADS) k_chain_hash(const uint32_t *__restrict__ tokens, int64_t n_tokens,
                                                            const int64_t *__restrict__ tok_off,
                                                            const uint32_t *__restrict__ s, int64_t R, uint64_t N,
                                                            uint64_t pos_base, uint32_t req_base,
                                                            uint64_t P_init, uint64_t *__restrict__ hash_out,
                                                            uint32_t *__restrict__ req_out,
                                                            uint32_t *__restrict__ key_out,
                                                            uint64_t *__restrict__ val_out) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * K1_WARPS;
  const uint64_t w = (uint64_t)blockIdx.x * K1_WARPS + (threadIdx.x >> 5);
  uint32_t bound = 0;
  if (lane < 2) {  // first request r with s[r] >= target
    uint64_t target = pos_base + ((w + lane) * N) / nw;
    int64_t lo = 0, hi = R;
    while (lo < hi) {
      int64_t m = (lo + hi) >> 1;
      if ((uint64_t)s[m] >= target) hi = m; else lo = m + 1;
    }
    bound = (uint32_t)lo;
  }
  const uint32_t rb = __shfl_sync(0xffffffffu, bound, 0), re = __shfl_sync(0xffffffffu, bound, 1);
  uint32_t key[16];
#pragma unroll
  for (int i = 0; i < 16; i++) key[i] = (uint32_t)fmix64((uint64_t)(i + 1));
  const uint64_t B0 = s[rb], B1 = s[re];
  const uint64_t RP = kChainR * P_init;
  uint64_t carry = 0;
  uint32_t r = rb;  // per-thread request cursor (monotone across rounds)
  for (uint64_t base = B0; base < B1; base += 32) {
    const uint64_t b = base + lane;
    const bool valid = b < B1;
    Aff e = {1, 0};
    uint32_t k = 0, sr = 0, n = 0;
    if (valid) {
      while (r + 1 < re && (uint64_t)s[r + 1] <= b) r++;
      sr = s[r];
      n = s[r + 1] - sr;
      k = (uint32_t)(b - sr);
      uint32_t t[16];
      load_block_tokens(tokens + tok_off[r] + 16 * (int64_t)k, tokens + n_tokens, t);
      uint64_t c = nh_block(t, key);
      e = (k == 0) ? Aff{0, RP + c} : Aff{kChainR, c};
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      uint64_t ua = __shfl_up_sync(0xffffffffu, e.a, off);
      uint64_t ub = __shfl_up_sync(0xffffffffu, e.b, off);
      if (lane >= off) e = aff_compose(Aff{ua, ub}, e);
    }
    const uint64_t P = e.a * carry + e.b;
    if (valid) {
      uint64_t j = (uint64_t)sr + n - 1 - k - pos_base;
      const uint64_t h = fmix64(P);
      hash_out[j] = h;
      req_out[j] = r + req_base;
      if (key_out) {  // K2's sort input, fused (k_sort_prep's mix): saves re-reading the hashes
        const uint64_t m = fmix64(h ^ kSortMixC);
        key_out[j] = (uint32_t)(m >> 32);
        val_out[j] = (m << 32) | (uint64_t)(uint32_t)j;
      }
    }
    carry = __shfl_sync(0xffffffffu, P, 31);  // last block of the round (beyond B1: unused)
  }
}

// HASHES mode: copy caller hashes into touch order (warp per request)
__global__ void k_copy_hashes(const uint64_t *__restrict__ bh, const int64_t *__restrict__ src_off,
                              const uint32_t *__restrict__ s, int64_t R, uint32_t pos_base, uint32_t req_base,
                              uint64_t *__restrict__ hash_out, uint32_t *__restrict__ req_out) {
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < R; r += nw) {
    uint32_t sr = s[r], n = s[r + 1] - sr;
    const uint64_t *src = bh + src_off[r];
    for (uint32_t k = lane; k < n; k += 32) {
      uint32_t j = sr + n - 1 - k - pos_base;
      hash_out[j] = src[k];
      req_out[j] = (uint32_t)r + req_base;
    }
  }
}

// ------------------------------------------------------------------ a3: K2 ----
__global__ void k_iota(uint32_t *v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)i;
}

// Sort key: a 32-bit fingerprint of the 64-bit hash (top half of a bijective mix m, so
// caller-provided structured hashes cannot crowd one key); value: (other half of m << 32) |
// position, so equality is decided on all 64 bits without gathers.
__global__ void k_sort_prep(const uint64_t *__restrict__ hash, uint64_t N, uint32_t *__restrict__ key,
                            uint64_t *__restrict__ val) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t m = fmix64(hash[j] ^ kSortMixC);  // bijection: (key, val >> 32) identifies h
    key[j] = (uint32_t)(m >> 32);
    val[j] = (m << 32) | (uint64_t)(uint32_t)j;
  }
}

// prev is assembled per bucket of 2^PB consecutive positions: every position appears exactly
// once among the (position, prev) pairs, so bucket b owns pair slots [b << PB, (b+1) << PB).
constexpr int PB = 11;

// In fingerprint-sorted order (stable: positions ascending within a key), the previous
// occurrence of element i is the nearest earlier element of its key run whose full hash
// matches (almost always i-1; a bounded scan, longer fingerprint-collision cases overflow).
constexpr int LINK_SCAN = 32;

// Each warp links LINK_U * 32 consecutive sorted elements: the predecessor element comes by
// shuffle, and the LINK_U slot reservations are issued before any result is consumed so their
// L2 round trips overlap.
constexpr int LINK_U = 4;
__global__ void __launch_bounds__(256) k_link_prev(const uint32_t *__restrict__ ks, const uint64_t *__restrict__ vs,
                                                   uint64_t N, unsigned *__restrict__ cursor, uint2 *__restrict__ pairs,
                                                   uint2 *__restrict__ ovf, uint32_t *__restrict__ n_ovf,
                                                   uint8_t *__restrict__ qf, uint8_t *__restrict__ nx) {
  const int lane = threadIdx.x & 31;
  const uint64_t nchunk = (N + 32 * LINK_U - 1) / (32 * LINK_U);
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; c < nchunk; c += nwarps) {
    const uint64_t i0 = c * 32 * LINK_U;
    uint32_t k[LINK_U], p[LINK_U], bk[LINK_U], same[LINK_U], base[LINK_U];
    uint64_t v[LINK_U];
    bool ovfl[LINK_U];
#pragma unroll
    for (int u = 0; u < LINK_U; u++) {
      const uint64_t i = i0 + u * 32 + lane;
      k[u] = i < N ? ks[i] : 0xFFFFFFFFu;
      v[u] = i < N ? vs[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < LINK_U; u++) {
      const uint64_t i = i0 + u * 32 + lane;
      uint32_t kq = __shfl_up_sync(0xFFFFFFFFu, k[u], 1);
      uint64_t vq = __shfl_up_sync(0xFFFFFFFFu, v[u], 1);
      if (lane == 0) {
        if (i > 0) { kq = ks[i - 1]; vq = vs[i - 1]; }
        else kq = ~k[u];
      }
      p[u] = kNone;
      ovfl[u] = false;
      uint64_t pred = ~0ull;  // sorted index of the previous occurrence
      if (i < N && kq == k[u]) {
        if ((vq >> 32) == (v[u] >> 32)) {
          p[u] = (uint32_t)vq;
          pred = i - 1;
        } else {  // fingerprint collision: bounded backward scan of the key run
          uint64_t t = i - 1;
          int steps = 1;
          for (; t > 0 && ks[t - 1] == k[u] && steps < LINK_SCAN; t--, steps++) {
            const uint64_t w = vs[t - 1];
            if ((w >> 32) == (v[u] >> 32)) { p[u] = (uint32_t)w; pred = t - 1; break; }
          }
          ovfl[u] = p[u] == kNone && steps == LINK_SCAN && t > 0 && ks[t - 1] == k[u];
        }
      }
      if (qf && i < N) {  // first-in-range flag (overflow: fixed by k_link_overflow), has-next mark
        qf[i] = p[u] == kNone ? 1 : 0;
        if (pred != ~0ull) nx[pred] = 1;
      }
    }
#pragma unroll
    for (int u = 0; u < LINK_U; u++) {
      const bool in = i0 + u * 32 + lane < N;
      bk[u] = in ? ((uint32_t)v[u] >> PB) : 0xFFFFFFFFu;
      same[u] = __match_any_sync(0xFFFFFFFFu, bk[u]);
      base[u] = 0;
      if (in && lane == __ffs(same[u]) - 1) base[u] = atomicAdd(&cursor[bk[u]], (unsigned)__popc(same[u]));
    }
#pragma unroll
    for (int u = 0; u < LINK_U; u++) {
      const uint64_t i = i0 + u * 32 + lane;
      const uint32_t b = __shfl_sync(0xFFFFFFFFu, base[u], __ffs(same[u]) - 1);
      if (i < N) {
        const uint32_t slot = (bk[u] << PB) + b + __popc(same[u] & ((1u << lane) - 1u));
        pairs[slot] = make_uint2((uint32_t)v[u], p[u]);
        if (ovfl[u]) ovf[atomicAdd(n_ovf, 1u)] = make_uint2((uint32_t)i, slot);  // resolved by k_link_overflow
      }
    }
  }
}

// Tile-staged variant (N <= 2^(12+P)): a CTA links a tile of 8192 consecutive sorted elements
// in two sweeps.  Sweep 1 histograms the tile's positions by 2^P-position bucket (shared-memory
// atomics); one block scan turns the histogram into tile-local offsets and ONE global atomic per
// (tile, bucket) reserves the bucket's run of pair slots.  Sweep 2 (the tile again, now from L2)
// links each element and stages its (position, prev) pair in shared memory grouped by bucket;
// the staged tile is then written out in order, so a warp's stores form runs of consecutive
// slots instead of 32 scattered 8-byte sectors.
constexpr int LT_THREADS = 1024, LT_U = 8, LT_TILE = LT_THREADS * LT_U;
constexpr int LT_MAX_BUCKETS = 4096;
template <int P>
__global__ void __launch_bounds__(LT_THREADS, 2) k_link_tile(const uint32_t *__restrict__ ks,
                                                          const uint64_t *__restrict__ vs, uint64_t N, int nbk,
                                                          unsigned *__restrict__ cursor, uint2 *__restrict__ pairs,
                                                          uint2 *__restrict__ ovf, uint32_t *__restrict__ n_ovf,
                                                          uint8_t *__restrict__ qf, uint8_t *__restrict__ nx) {
  typedef cub::BlockScan<uint32_t, LT_THREADS> Scan;
  __shared__ typename Scan::TempStorage scan_ts;
  extern __shared__ __align__(16) uint8_t lt_raw[];
  uint2 *stage = reinterpret_cast<uint2 *>(lt_raw);                       // [LT_TILE]
  uint32_t *cur = reinterpret_cast<uint32_t *>(lt_raw + 8 * LT_TILE);     // [nbk]
  int32_t *off = reinterpret_cast<int32_t *>(cur + nbk);                  // [nbk]
  const int lane = threadIdx.x & 31;
  const uint64_t ntile = (N + LT_TILE - 1) / LT_TILE;
  const int per = (nbk + LT_THREADS - 1) / LT_THREADS;
  for (uint64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const uint64_t t0 = tile * LT_TILE;
    const uint32_t tn = (uint32_t)(N - t0 < (uint64_t)LT_TILE ? N - t0 : LT_TILE);
    for (int b = threadIdx.x; b < nbk; b += LT_THREADS) cur[b] = 0;
    __syncthreads();
    // sweep 1: bucket histogram of the tile's positions
#pragma unroll
    for (int u = 0; u < LT_U; u++) {
      const uint32_t q = u * LT_THREADS + threadIdx.x;
      if (q < tn) atomicAdd(&cur[(uint32_t)vs[t0 + q] >> P], 1u);
    }
    __syncthreads();
    // tile-local exclusive offsets; one global reservation per non-empty bucket
    uint32_t part = 0;
    for (int e = 0; e < per; e++) {
      const int b = threadIdx.x * per + e;
      if (b < nbk) part += cur[b];
    }
    uint32_t run;
    Scan(scan_ts).ExclusiveSum(part, run);
    constexpr int PER_MAX = LT_MAX_BUCKETS / LT_THREADS;
    uint32_t cc[PER_MAX], gg[PER_MAX];
#pragma unroll
    for (int e = 0; e < PER_MAX; e++) {  // all reservations in flight before any result is used
      const int b = threadIdx.x * per + e;
      cc[e] = (e < per && b < nbk) ? cur[b] : 0u;
      gg[e] = cc[e] ? atomicAdd(&cursor[b], cc[e]) : 0u;
    }
#pragma unroll
    for (int e = 0; e < PER_MAX; e++) {
      const int b = threadIdx.x * per + e;
      if (e < per && b < nbk) {
        off[b] = (int32_t)gg[e] - (int32_t)run;
        cur[b] = run;
        run += cc[e];
      }
    }
    __syncthreads();
    // sweep 2: link and stage grouped by bucket
#pragma unroll 2
    for (int u = 0; u < LT_U; u++) {
      const uint32_t q = u * LT_THREADS + threadIdx.x;
      const uint64_t i = t0 + q;
      const bool in = q < tn;
      const uint32_t k = in ? ks[i] : 0xFFFFFFFFu;
      const uint64_t v = in ? vs[i] : 0;
      uint32_t kq = __shfl_up_sync(0xFFFFFFFFu, k, 1);
      uint64_t vq = __shfl_up_sync(0xFFFFFFFFu, v, 1);
      if (lane == 0) {
        if (in && i > 0) { kq = ks[i - 1]; vq = vs[i - 1]; }
        else kq = ~k;
      }
      if (in) {
        uint32_t p = kNone;
        bool ov = false;
        uint64_t pred = ~0ull;
        if (kq == k) {
          if ((vq >> 32) == (v >> 32)) {
            p = (uint32_t)vq;
            pred = i - 1;
          } else {  // fingerprint collision: bounded backward scan of the key run
            uint64_t t = i - 1;
            int steps = 1;
            for (; t > 0 && ks[t - 1] == k && steps < LINK_SCAN; t--, steps++) {
              const uint64_t w = vs[t - 1];
              if ((w >> 32) == (v >> 32)) { p = (uint32_t)w; pred = t - 1; break; }
            }
            ov = p == kNone && steps == LINK_SCAN && t > 0 && ks[t - 1] == k;
          }
        }
        if (qf) {
          qf[i] = p == kNone ? 1 : 0;
          if (pred != ~0ull) nx[pred] = 1;
        }
        const uint32_t j = (uint32_t)v, bk = j >> P;
        const uint32_t loc = atomicAdd(&cur[bk], 1u);
        stage[loc] = make_uint2(j, p);
        if (ov) ovf[atomicAdd(n_ovf, 1u)] = make_uint2((uint32_t)i, (uint32_t)((bk << P) + off[bk] + (int32_t)loc));
      }
    }
    __syncthreads();
    // write the staged tile out in order: runs of consecutive slots per bucket
    for (uint32_t q = threadIdx.x; q < tn; q += LT_THREADS) {
      const uint2 e = stage[q];
      const uint32_t bk = e.x >> P;
      pairs[(uint64_t)(bk << P) + (int64_t)off[bk] + q] = e;
    }
    __syncthreads();
  }
}

// Rare slow path (32-bit fingerprint collisions in long key runs): one CTA per overflowed
// element walks the key run backwards 1024 elements per step; the largest matching position
// below i is the previous occurrence.
constexpr int OVF_THREADS = 1024;
__global__ void __launch_bounds__(OVF_THREADS) k_link_overflow(const uint32_t *__restrict__ ks,
                                                                const uint64_t *__restrict__ vs,
                                                                const uint2 *__restrict__ ovf,
                                                                const uint32_t *__restrict__ n_ovf,
                                                                uint2 *__restrict__ pairs, uint8_t *__restrict__ qf,
                                                                uint8_t *__restrict__ nx) {
  __shared__ unsigned long long best1;  // 1 + best sorted index, 0 = none
  __shared__ int ended;
  const uint32_t n = *n_ovf;
  for (uint32_t w = blockIdx.x; w < n; w += gridDim.x) {
    const uint2 o = ovf[w];
    const uint64_t i = o.x;
    const uint32_t k = ks[i];
    const uint64_t hi = vs[i] >> 32;
    if (threadIdx.x == 0) { best1 = 0; ended = 0; }
    __syncthreads();
    for (int64_t base = (int64_t)i - 1 - LINK_SCAN; base >= 0; base -= OVF_THREADS) {
      int64_t t = base - threadIdx.x;
      bool in = t >= 0 && ks[t] == k;
      if (!in) atomicOr(&ended, 1);
      else if ((vs[t] >> 32) == hi) atomicMax(&best1, (unsigned long long)t + 1);
      __syncthreads();
      bool stop = best1 != 0 || ended;
      __syncthreads();
      if (stop) break;
    }
    if (threadIdx.x == 0) {
      pairs[o.y].y = best1 ? (uint32_t)vs[best1 - 1] : kNone;
      if (qf && best1) { qf[i] = 0; nx[best1 - 1] = 1; }
    }
    __syncthreads();
  }
}

// bucket b's pairs -> the 2^P-entry slice of prev[] in shared memory -> one coalesced write
// (sl > 0: bucket b's pairs sit in 2^sl sub-regions of 2^(P-sl) by position mod 2^sl; a partial
// last bucket fills a prefix of each sub-region)
template <int P>
__global__ void __launch_bounds__(1024) k_bucket_assemble(const uint2 *__restrict__ pairs, uint64_t N,
                                                           uint32_t *__restrict__ prev, uint32_t sl) {
  extern __shared__ uint32_t slice[];
  const uint64_t nb = (N + (1u << P) - 1) >> P;
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint64_t lo = b << P;
    const uint32_t cnt = (uint32_t)((N - lo) < (1u << P) ? (N - lo) : (1u << P));
    const bool part = cnt < (1u << P) && sl > 0;
    const uint32_t span = part ? (1u << P) : cnt;
    for (uint32_t q0 = 0; q0 < span; q0 += 8 * blockDim.x) {  // 8 loads in flight per thread
      uint2 pr[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const uint32_t q = q0 + e * blockDim.x + threadIdx.x;
        bool ok = q < span;
        if (part && ok)  // sub-region q >> (P - sl) holds (cnt + 2^sl - 1 - sub) >> sl pairs
          ok = (q & ((1u << (P - sl)) - 1u)) < ((cnt + (1u << sl) - 1u - (q >> (P - sl))) >> sl);
        pr[e] = ok ? pairs[lo + q] : make_uint2(0xFFFFFFFFu, 0);
      }
#pragma unroll
      for (int e = 0; e < 8; e++)
        if (pr[e].x != 0xFFFFFFFFu) slice[pr[e].x & ((1u << P) - 1)] = pr[e].y;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < cnt; q += blockDim.x) prev[lo + q] = slice[q];
    __syncthreads();
  }
}

__device__ __forceinline__ void warp_count_add(uint32_t *arr, uint32_t key, bool pred) {
  unsigned active = __activemask();
  unsigned pm = __ballot_sync(active, pred);
  if (!pred) return;
  unsigned same = __match_any_sync(pm, key);
  if ((__ffs(same) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&arr[key], (uint32_t)__popc(same));
}

__global__ void k_access_info(uint64_t N, const uint32_t *__restrict__ prev, const uint32_t *__restrict__ req,
                              const uint32_t *__restrict__ s, const int64_t *__restrict__ arr,
                              const uint64_t *__restrict__ hash, uint32_t *__restrict__ delta,
                              uint32_t *__restrict__ first_cnt, uint32_t *__restrict__ reuse_cnt,
                              uint8_t *__restrict__ run_flag, LoadStats *st) {
  unsigned flags = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t p = prev[j], r = req[j];
    uint32_t dl = kNone;
    if (p != kNone) {
      uint32_t rp = req[p];
      int64_t d = arr[r] - arr[rp];
      if (d < 0 || d >= (int64_t)kNone) flags |= F_DELTA; else dl = (uint32_t)d;
      uint32_t kj = s[r + 1] - 1 - (uint32_t)j;
      uint32_t kp = s[rp + 1] - 1 - p;
      if (kj != kp) flags |= F_CHAIN;
      // parents must match (R7); when the parent access links to p + 1 the K2 link already
      // proves equal hashes (the common case inside a run), so only run ends gather hashes
      else if (kj > 0 && prev[j + 1] != p + 1 && hash[j + 1] != hash[p + 1]) flags |= F_CHAIN;
    }
    delta[j] = dl;
    // K3 run heads: a reuse access whose predecessor position is not its previous position
    // plus one, or the first position of its request (stack_depth.cu)
    uint8_t head = 0;
    if (p != kNone) {
      uint32_t pm = j > 0 ? prev[j - 1] : kNone;
      head = ((uint32_t)j == s[r] || pm == kNone || p != pm + 1) ? 1 : 0;
    }
    run_flag[j] = head;
    warp_count_add(first_cnt, r, p == kNone);
    warp_count_add(reuse_cnt, r, p != kNone);
  }
  if (flags) atomicOr(&st->flags, flags);
}

// Whole traces, K2 per access (round 2): the run-head flags of K3 and the per-request first /
// reuse counts; first accesses get delta = none.  The reuse interval and the chain checks of a
// reuse access are the same for every access of its run (one earlier request, chain positions
// falling together), so k_run_delta computes them once per run.  A first access right after a
// reuse access of its request breaks R7 by itself (the reused block's parent was never seen).
__global__ void k_access_flags(uint64_t N, const uint32_t *__restrict__ prev, const uint32_t *__restrict__ req,
                               const uint32_t *__restrict__ s, uint32_t *__restrict__ delta,
                               uint8_t *__restrict__ run_flag, LoadStats *st) {
  unsigned flags = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < N; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = prev[j], r = req[j];
    const uint32_t pm = j > 0 ? prev[j - 1] : kNone;
    const bool start = (uint32_t)j == s[r];
    uint8_t head = 0;
    if (p != kNone) head = (start || pm == kNone || p != pm + 1) ? 1 : 0;
    else {
      delta[j] = kNone;
      if (!start && pm != kNone) flags |= F_CHAIN;
    }
    run_flag[j] = head;
  }
  if (flags) atomicOr(&st->flags, flags);
}

// per request: first accesses = blocks - reuse accesses (the runs' lengths, k_run_delta)
__global__ void k_first_from_reuse(int64_t R, const uint32_t *__restrict__ s, const uint32_t *__restrict__ reuse_cnt,
                                   uint32_t *__restrict__ first_cnt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x)
    first_cnt[r] = (s[r + 1] - s[r]) - reuse_cnt[r];
}

// Per run (a warp loads 32 runs' data at once): delta = arr[r] - arr[req[p0]] (R5), chain
// positions equal at the run's start (then along the run), the parent hashes equal at its end
// (inside a run the parent access links to p + 1, which the exact link proves equal); the run's
// delta is then written by all lanes, run after run.
__global__ void __launch_bounds__(256) k_run_delta(const int *__restrict__ m_ptr, const uint32_t *__restrict__ run_start,
                                                   const uint32_t *__restrict__ run_req,
                                                   const uint32_t *__restrict__ run_len,
                                                   const uint32_t *__restrict__ run_p0, const uint32_t *__restrict__ prev,
                                                   const uint32_t *__restrict__ req, const uint32_t *__restrict__ s,
                                                   const int64_t *__restrict__ arr, const uint64_t *__restrict__ hash,
                                                   uint32_t *__restrict__ delta, uint32_t *__restrict__ reuse_cnt,
                                                   LoadStats *st) {
  const int M = *m_ptr;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  unsigned flags = 0;
  for (int q0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; q0 < M; q0 += nw * 32) {
    const int q = q0 + lane;
    uint32_t j0 = 0, L = 0, dl = kNone;
    if (q < M) {
      j0 = run_start[q];
      L = run_len[q];
      const uint32_t r = run_req[q], p0 = run_p0[q];
      atomicAdd(&reuse_cnt[r], L);  // every reuse access lies in exactly one run
      const uint32_t rp = req[p0];
      const int64_t d = arr[r] - arr[rp];
      if (d < 0 || d >= (int64_t)kNone) flags |= F_DELTA; else dl = (uint32_t)d;
      const uint32_t kj = s[r + 1] - 1 - j0, kp = s[rp + 1] - 1 - p0;
      if (kj != kp) flags |= F_CHAIN;
      else {
        const uint32_t je = j0 + L - 1, pe = p0 + L - 1;  // the run's last access (chain position kj - L + 1)
        if (kj - (L - 1) > 0 && prev[je + 1] != pe + 1 && hash[je + 1] != hash[pe + 1]) flags |= F_CHAIN;
      }
    }
    const int nk = M - q0 < 32 ? M - q0 : 32;
    for (int k = 0; k < nk; k++) {
      const uint32_t jk = __shfl_sync(0xFFFFFFFFu, j0, k), Lk = __shfl_sync(0xFFFFFFFFu, L, k);
      const uint32_t dk = __shfl_sync(0xFFFFFFFFu, dl, k);
      for (uint32_t t = lane; t < Lk; t += 32) delta[jk + t] = dk;
    }
  }
  if (flags) atomicOr(&st->flags, flags);
}

// groups: requests with at least one block, keyed by their root hash (block k = 0, the
// last touch of the request)
// (s points at the first request considered; hash is indexed by position - pos_base)
__global__ void k_root_keys(int64_t R, const uint32_t *__restrict__ s, const uint64_t *__restrict__ hash,
                            uint32_t pos_base, uint64_t *__restrict__ key, uint32_t *__restrict__ val,
                            uint8_t *__restrict__ flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
    bool has = s[r + 1] > s[r];
    flag[r] = has;
    key[r] = has ? hash[s[r + 1] - 1 - pos_base] : 0;
    val[r] = (uint32_t)r;
  }
}

__global__ void k_run_heads(const uint64_t *__restrict__ key, const int *__restrict__ m_ptr, uint32_t *__restrict__ head) {
  int m = *m_ptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

__global__ void k_run_reuse(const uint32_t *__restrict__ val, const uint32_t *__restrict__ run_incl,
                            const int *__restrict__ m_ptr, const uint32_t *__restrict__ reuse_cnt,
                            unsigned long long *__restrict__ run_reuse, uint32_t *__restrict__ n_runs) {
  int m = *m_ptr;
  // runs are contiguous in sorted order, so a warp's lanes mostly share a run: reduce per run
  // inside the warp first (hot system-prompt roots would otherwise serialise on one address)
  const int m_pad = (m + 31) & ~31;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m_pad; i += gridDim.x * blockDim.x) {
    const bool in = i < m;
    const uint32_t rid = in ? run_incl[i] - 1 : 0xFFFFFFFFu;
    const uint32_t v = in ? reuse_cnt[val[i]] : 0u;
    const unsigned same = __match_any_sync(0xFFFFFFFFu, rid);
    const uint32_t sum = __reduce_add_sync(same, v);
    if (in && (int)(threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&run_reuse[rid], (unsigned long long)sum);
    if (i == m - 1) *n_runs = run_incl[i];
  }
}

__global__ void k_rank_keys(const unsigned long long *__restrict__ run_reuse, const uint32_t *__restrict__ n_runs,
                            uint64_t *__restrict__ key, uint32_t *__restrict__ idx, uint32_t cap) {
  uint32_t n = *n_runs;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
    // runs are in ascending root-hash order; a stable sort by ~reuse gives (reuse desc, hash asc)
    key[i] = i < n ? ~(uint64_t)run_reuse[i] : ~0ull;
    idx[i] = i;
  }
}

__global__ void k_rank_of_run(const uint32_t *__restrict__ ranked, const uint32_t *__restrict__ n_runs,
                              uint32_t *__restrict__ rank) {
  uint32_t n = *n_runs;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rank[ranked[i]] = i;
}

__global__ void k_assign_groups(const uint32_t *__restrict__ val, const uint32_t *__restrict__ run_incl,
                                const int *__restrict__ m_ptr, const uint32_t *__restrict__ rank, int K,
                                uint16_t *__restrict__ grp) {
  int m = *m_ptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    uint32_t rk = rank[run_incl[i] - 1];
    grp[val[i]] = (uint16_t)(rk < (uint32_t)K ? rk : (uint32_t)K);
  }
}

__global__ void k_fill_u16(uint16_t *p, int64_t n, uint16_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// requests [r_base, r_base + R): grp is global, first_cnt / reuse_cnt local
__global__ void k_group_tables(int64_t R, uint32_t r_base, const uint16_t *__restrict__ grp,
                               const uint32_t *__restrict__ first_cnt, const uint32_t *__restrict__ reuse_cnt,
                               unsigned long long *__restrict__ tab, int G) {
  // tab[2g] = U_g, tab[2g+1] = reuse_g; privatised per block in smem (G <= 1024)
  extern __shared__ unsigned long long ts[];
  for (int i = threadIdx.x; i < 2 * G; i += blockDim.x) ts[i] = 0;
  __syncthreads();
  // few groups, many requests: reduce within the warp per group first (match_any), then one
  // shared-memory atomic per (warp, group)
  const int64_t Rp = (R + 31) & ~(int64_t)31;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < Rp; r += (int64_t)gridDim.x * blockDim.x) {
    const bool in = r < R;
    const int g = in ? grp[r_base + r] : -1;
    const uint32_t fc = in ? first_cnt[r] : 0u, rc = in ? reuse_cnt[r] : 0u;
    const unsigned same = __match_any_sync(0xFFFFFFFFu, g);
    const uint32_t fs = __reduce_add_sync(same, fc), rs = __reduce_add_sync(same, rc);
    if (in && (int)(threadIdx.x & 31) == __ffs(same) - 1) {
      if (fs) atomicAdd(&ts[2 * g], (unsigned long long)fs);
      if (rs) atomicAdd(&ts[2 * g + 1], (unsigned long long)rs);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * G; i += blockDim.x)
    if (ts[i]) atomicAdd(&tab[i], ts[i]);
}

// K2's sort policy on sm_100: CUB onesweep, 8-bit digits, 256 threads x 32 items, 32-bit
// offsets (N < 2^32 is enforced at load).  Measured on the K2 shape (1.06e8 u32 keys + u64
// values): 3.53 ms vs 3.64 ms for CUB's default tuning (tools/sort_policy_bench.cu).
struct K2SortHub {
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = 8;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, uint32_t, 8>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, 8>;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<256, 32, uint64_t, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, 8>;
    // never used on sm_100 (onesweep), required by the dispatcher's instantiation
    using ScanPolicy = cub::AgentScanPolicy<512, 23, uint32_t, cub::BLOCK_LOAD_WARP_TRANSPOSE, cub::LOAD_DEFAULT,
                                            cub::BLOCK_STORE_WARP_TRANSPOSE, cub::BLOCK_SCAN_RAKING_MEMOIZE>;
    using DownsweepPolicy = cub::AgentRadixSortDownsweepPolicy<512, 23, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                               cub::LOAD_DEFAULT, cub::RADIX_RANK_MATCH,
                                                               cub::BLOCK_SCAN_WARP_SCANS, 7>;
    using AltDownsweepPolicy = cub::AgentRadixSortDownsweepPolicy<256, 47, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                                  cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                                  cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using UpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 23, uint64_t, cub::LOAD_DEFAULT, 7>;
    using AltUpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 47, uint64_t, cub::LOAD_DEFAULT, 6>;
    using SingleTilePolicy = cub::AgentRadixSortDownsweepPolicy<256, 19, uint64_t, cub::BLOCK_LOAD_DIRECT,
                                                                cub::LOAD_LDG, cub::RADIX_RANK_MEMOIZE,
                                                                cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using SegmentedPolicy = cub::AgentRadixSortDownsweepPolicy<192, 39, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                               cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                               cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using AltSegmentedPolicy = cub::AgentRadixSortDownsweepPolicy<384, 11, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                                  cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                                  cub::BLOCK_SCAN_WARP_SCANS, 5>;
  };
  using MaxPolicy = Policy1000;
};
using K2Sort = cub::DispatchRadixSort<false, uint32_t, uint64_t, uint32_t, K2SortHub>;

// ------------------------------------------------------------------ driver ----
template <typename T>
static kareto_status to_device(kareto_ctx *ctx, const T *src, size_t n, bool on_device, DBuf<T> &own,
                               const T **out) {
  if (on_device || n == 0) {
    *out = src;
    return KARETO_OK;
  }
  KTRY(own.alloc(ctx, n));
  KCUDA(ctx, cudaMemcpyAsync(own.p, src, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  *out = own.p;
  return KARETO_OK;
}

kareto_status ingest(kareto_ctx *ctx, const kareto_trace_desc *d, kareto_trace *tr, Ingest &in) {
  const int64_t R = d->n_requests;
  if (R < 1) return fail(ctx, KARETO_E_INVALID, "n_requests must be >= 1");
  if (R >= (int64_t)kNone) return fail(ctx, KARETO_E_OVERFLOW, "too many requests");
  if (d->top_k < 0 || d->top_k > 1023) return fail(ctx, KARETO_E_INVALID, "top_k must be in [0, 1023]");
  if (d->mode != KARETO_TOKENS && d->mode != KARETO_HASHES) return fail(ctx, KARETO_E_INVALID, "bad mode");
  if (!d->arrival_ms || !d->output_tokens || !d->offsets) return fail(ctx, KARETO_E_INVALID, "null trace array");
  const bool dev = d->inputs_on_device != 0;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;

  // total elements of the token / hash array (offsets[R])
  int64_t total = 0;
  if (dev) KCUDA(ctx, cudaMemcpyAsync(&total, d->offsets + R, 8, cudaMemcpyDeviceToHost, st));
  else total = d->offsets[R];
  KCUDA(ctx, cudaStreamSynchronize(st));
  if (total < 0) return fail(ctx, KARETO_E_PARSE, "offsets[R] < 0");
  if (d->mode == KARETO_TOKENS && total > 0 && !d->tokens) return fail(ctx, KARETO_E_INVALID, "tokens is null");
  if (d->mode == KARETO_HASHES && total > 0 && !d->block_hash) return fail(ctx, KARETO_E_INVALID, "block_hash null");
  in.total = total;
  {
    Pass ps(ctx, "h2d", 0, 0);
    KTRY(to_device(ctx, d->arrival_ms, R, dev, in.h_arr, &in.arrival));
    KTRY(to_device(ctx, d->output_tokens, R, dev, in.h_out, &in.out_tok));
    KTRY(to_device(ctx, d->offsets, R + 1, dev, in.h_off, &in.offsets));
    if (d->mode == KARETO_HASHES && d->input_tokens)
      KTRY(to_device(ctx, d->input_tokens, R, dev, in.h_in, &in.input_tokens));
  }
  tr->R = R;
  tr->K = d->top_k;

  DBuf<uint8_t> tmp;
  KTRY(in.stats.alloc(ctx, 1));
  KTRY(in.stats.zero());
  DBuf<uint64_t> skey, skey2, s64;
  DBuf<uint32_t> sidx, order;
  DBuf<int64_t> arr_sorted;
  KTRY(skey.alloc(ctx, R)); KTRY(skey2.alloc(ctx, R)); KTRY(sidx.alloc(ctx, R)); KTRY(order.alloc(ctx, R));
  KTRY(arr_sorted.alloc(ctx, R)); KTRY(in.src_off.alloc(ctx, R)); KTRY(in.nblk.alloc(ctx, R + 1));
  KTRY(s64.alloc(ctx, R + 1));
  int key_bits = 64;
  {
    Pass ps(ctx, "a1_sort_keys", 1, 2);
    DBuf<unsigned long long> mnmx;
    KTRY(mnmx.alloc(ctx, 2));
    const unsigned long long init[2] = {~0ull, 0ull};
    KCUDA(ctx, cudaMemcpyAsync(mnmx.p, init, 16, cudaMemcpyHostToDevice, st));
    k_sort_keys<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(in.arrival, R, skey.p, sidx.p, mnmx.p);
    k_rebase_keys<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(skey.p, R, mnmx.p);
    unsigned long long h[2];
    KCUDA(ctx, cudaMemcpyAsync(h, mnmx.p, 16, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    const uint64_t span = h[1] - h[0];
    key_bits = 1;
    while (key_bits < 64 && (span >> key_bits) != 0) key_bits++;
  }
  {
    Pass ps(ctx, "a1_sort_requests", 0, 1);
    KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, skey.p, skey2.p, sidx.p, order.p, (int)R, 0, key_bits, st);
    }));
  }
  KCUDA(ctx, cudaMemsetAsync(in.nblk.p + R, 0, 8, st));
  KMALLOC(ctx, tr->inlen, 4 * (size_t)R, st);
  KMALLOC(ctx, tr->outlen, 4 * (size_t)R, st);
  {
    Pass ps(ctx, "a1_req_meta", 1, 1);
    k_req_meta<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(R, d->mode, order.p, in.arrival, in.out_tok, in.offsets,
                                                          in.input_tokens, arr_sorted.p, in.src_off.p, in.nblk.p,
                                                          tr->inlen, tr->outlen, in.stats.p);
  }
  {
    Pass ps(ctx, "a1_scan_starts", 0, 1);
    KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceScan::ExclusiveSum(t, b, in.nblk.p, s64.p, (int)(R + 1), st);
    }));
  }
  KMALLOC(ctx, tr->s, 4 * (size_t)(R + 1), st);
  {
    Pass ps(ctx, "a1_narrow", 1, 1);
    k_narrow_starts<<<grid_for(R + 1, 256, 4 * sms), 256, 0, st>>>(R, s64.p, tr->s, arr_sorted.p, in.stats.p);
  }
  LoadStats &hs = in.hs;
  KCUDA(ctx, cudaMemcpyAsync(&hs, in.stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaStreamSynchronize(st));
  if (hs.flags & F_OFFSETS) return fail(ctx, KARETO_E_PARSE, "offsets are not nondecreasing");
  if (hs.flags & F_OUTPUT) return fail(ctx, KARETO_E_PARSE, "output_tokens < 0");
  if (hs.flags & F_INPUT_LEN) return fail(ctx, KARETO_E_PARSE, "input_tokens < 16 * blocks (or absurd length)");
  const uint64_t N = hs.n_total;
  if (N >= (uint64_t)kNone - 1) return fail(ctx, KARETO_E_OVERFLOW, "%llu block accesses >= 2^32-2", (unsigned long long)N);
  tr->N = (int64_t)N;
  tr->max_blocks = (int32_t)hs.max_blocks;
  tr->span_ms = hs.arr_last - hs.arr_first;
  if (tr->span_ms < 1) tr->span_ms = 1;
  tr->O = hs.O;
  tr->SL = ((unsigned __int128)hs.sl_hi << 32) + hs.sl_lo;
  tr->SQ = ((unsigned __int128)hs.sq_hi << 32) + hs.sq_lo;
  if (tr->SL > (unsigned __int128)UINT64_MAX) return fail(ctx, KARETO_E_OVERFLOW, "sum of input tokens >= 2^64");
  tr->Ltok = (uint64_t)tr->SL;
  tr->arr = arr_sorted.detach();
  KMALLOC(ctx, tr->grp, 2 * (size_t)R, st);
  return KARETO_OK;
}

kareto_status upload_payload(kareto_ctx *ctx, const kareto_trace_desc *d, int64_t lo, int64_t hi,
                             DBuf<uint32_t> &tok, DBuf<uint64_t> &bh, const uint32_t **tok_base,
                             const uint64_t **bh_base) {
  *tok_base = nullptr;
  *bh_base = nullptr;
  const bool tokens = d->mode == KARETO_TOKENS;
  if (d->inputs_on_device || hi <= lo) {
    *tok_base = tokens ? d->tokens : nullptr;
    *bh_base = tokens ? nullptr : d->block_hash;
    return KARETO_OK;
  }
  Pass ps(ctx, "h2d", 0, 0);
  const size_t n = (size_t)(hi - lo);
  (void)tok;
  (void)bh;
  const size_t bytes = (tokens ? 4 : 8) * n;
  if (ctx->h2d_scratch_bytes < bytes) {  // the per-context staging buffer, grown on demand
    if (ctx->h2d_scratch) cudaFreeAsync(ctx->h2d_scratch, ctx->stream);
    ctx->h2d_scratch = nullptr;
    ctx->h2d_scratch_bytes = 0;
    KMALLOC(ctx, ctx->h2d_scratch, bytes, ctx->stream);
    ctx->h2d_scratch_bytes = bytes;
  }
  if (tokens) {
    uint32_t *p = static_cast<uint32_t *>(ctx->h2d_scratch);
    KCUDA(ctx, cudaMemcpyAsync(p, d->tokens + lo, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *tok_base = p - lo;
  } else {
    uint64_t *p = static_cast<uint64_t *>(ctx->h2d_scratch);
    KCUDA(ctx, cudaMemcpyAsync(p, d->block_hash + lo, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *bh_base = p - lo;
  }
  return KARETO_OK;
}

kareto_status chain_hash(kareto_ctx *ctx, const kareto_trace_desc *d, const kareto_trace *tr, const Ingest &in,
                         const uint32_t *tok_base, const uint64_t *bh_base, int64_t tok_end, int64_t r0, int64_t r1,
                         uint64_t *hash_out, uint32_t *req_out, SortedHashes *prep) {
  uint32_t se[2] = {0, (uint32_t)tr->N};
  if (!(r0 == 0 && r1 == tr->R && !tr->sharded)) {  // a whole trace's range is [0, N): no round trip
    KCUDA(ctx, cudaMemcpyAsync(&se[0], tr->s + r0, 4, cudaMemcpyDeviceToHost, ctx->stream));
    KCUDA(ctx, cudaMemcpyAsync(&se[1], tr->s + r1, 4, cudaMemcpyDeviceToHost, ctx->stream));
    KCUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const uint64_t n = (uint64_t)(se[1] - se[0]);
  if (n == 0) return KARETO_OK;
  const int sms = ctx->num_sms;
  if (d->mode == KARETO_TOKENS) {
    uint64_t P_init = fmix64(d->salt ^ kSaltC);
    // ~2048 blocks per warp, at least 16 warps per SM
    uint64_t nwarps = (n + 2047) / 2048;
    if (nwarps < (uint64_t)(16 * sms)) nwarps = 16 * sms;
    unsigned g = (unsigned)((nwarps + K1_WARPS - 1) / K1_WARPS);
    if (prep) {  // K2's sort input written by K1 (k_sort_prep fused)
      KTRY(prep->key.alloc(ctx, n));
      KTRY(prep->val.alloc(ctx, n));
    }
    Pass ps(ctx, "K1_chain_hash", 1, 1);
    k_chain_hash<<<g, K1_THREADS, 0, ctx->stream>>>(tok_base, tok_end, in.src_off.p + r0, tr->s + r0, r1 - r0, n,
                                                    se[0], (uint32_t)r0, P_init, hash_out, req_out,
                                                    prep ? prep->key.p : nullptr, prep ? prep->val.p : nullptr);
  } else {
    Pass ps(ctx, "K1_copy_hashes", 1, 1);
    k_copy_hashes<<<grid_for(32 * (r1 - r0), 256, 8 * sms), 256, 0, ctx->stream>>>(
        bh_base, in.src_off.p + r0, tr->s + r0, r1 - r0, se[0], (uint32_t)r0, hash_out, req_out);
  }
  return KARETO_OK;
}

// The bucket path of link_prev (bucket_link.cuh): sort (key, value) by the top BL_BITS key bits
// (stable), bucket bounds, chunks, k_bucket_link, k_bucket_fixup, k_bucket_assemble.  *ok = false
// if a table overflowed (nothing in prev is valid then).  The pending / last-position records
// use the unsorted input buffers (free after the sort) and a per-context scratch kept between
// loads (12 B per access), so a step does not map fresh gigabytes from the pool.
static kareto_status bucket_link(kareto_ctx *ctx, DBuf<uint32_t> &k32, DBuf<uint64_t> &v64, DBuf<uint32_t> &k32s,
                                 DBuf<uint64_t> &v64s, uint64_t N, uint32_t *prev, DBuf<uint8_t> &tmp, unsigned *ovf_dev) {
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  HostMarks hm("K2 bucket");
  {
    Pass ps(ctx, "K2_sort_buckets", 0, 1);
    cub::DoubleBuffer<uint32_t> dk(k32.p, k32s.p);
    cub::DoubleBuffer<uint64_t> dv(v64.p, v64s.p);
    KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
      return K2Sort::Dispatch(t, b, dk, dv, (uint32_t)N, 32 - BL_BITS, 32, true, st);
    }));
    if (dk.Current() != k32s.p) {
      std::swap(k32.p, k32s.p);
      std::swap(v64.p, v64s.p);
    }
  }
  hm.mark(st, "sort");
  DBuf<uint32_t> bstart, nch, cstart;
  DBuf<unsigned> ctr;
  KTRY(bstart.alloc(ctx, BL_NB + 1)); KTRY(nch.alloc(ctx, BL_NB + 1)); KTRY(cstart.alloc(ctx, BL_NB + 1));
  KTRY(ctr.alloc(ctx, 2)); KTRY(ctr.zero());
  {
    Pass ps(ctx, "K2_bucket_bounds", 1, 2);
    k_bucket_bounds_bs<<<(BL_NB + 1 + 255) / 256, 256, 0, st>>>(k32s.p, N, bstart.p);
    k_bucket_chunks<<<BL_NB / 256, 256, 0, st>>>(bstart.p, nch.p);
  }
  KCUDA(ctx, cudaMemsetAsync(nch.p + BL_NB, 0, 4, st));
  KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, nch.p, cstart.p, BL_NB + 1, st);
  }));
  DBuf<uint16_t> cbucket;  // chunk -> bucket (BL_BITS = 16)
  // no host round trip: the kernels read the chunk count from cstart[2^16]; rec_n is sized for
  // the most chunks N accesses can form
  const uint64_t max_chunks = (uint64_t)BL_NB + N / BL_CHUNK + 1;
  constexpr int PBT = 15;
  const uint64_t nbk = (N + (1u << PBT) - 1) >> PBT;
  // the pairs (8 B per access) and the last-position records (12 B) live in a per-context scratch
  // kept between loads: allocating ~2 GB from the stream-ordered pool at this point of every load
  // blocked the host for 4-6 ms (the pool reclaims pending frees), the device idling meanwhile
  DBuf<unsigned> cursor;
  DBuf<uint32_t> rec_n;
  uint32_t sl = BL_SUB_LOG2, cstride = BL_CSTRIDE;
  if (const char *e = getenv("KARETO_BL_SUB")) sl = (uint32_t)atoi(e) <= 8 ? (uint32_t)atoi(e) : 0u;
  if (const char *e = getenv("KARETO_BL_CSTRIDE")) cstride = (uint32_t)atoi(e) > 0 ? (uint32_t)atoi(e) : 1u;
  KTRY(cursor.alloc(ctx, (nbk << sl) * cstride)); KTRY(cursor.zero());
  KTRY(rec_n.alloc(ctx, 2 * max_chunks));
  KTRY(cbucket.alloc(ctx, max_chunks));
  k_chunk_bucket<<<BL_NB / 256, 256, 0, st>>>(cstart.p, cbucket.p);
  ctx->own_launches++;
  uint64_t *rec_m = v64.p, *lst_m = nullptr;  // the unsorted input buffers are free now
  uint32_t *rec_p = k32.p, *lst_p = nullptr;
  const size_t npairs = (size_t)nbk << PBT;  // padded: a partial last bucket fills sub-region prefixes
  const size_t need = 8 * npairs + 12 * (size_t)N + 512;
  if (ctx->k2_scratch_bytes < need) {
    if (ctx->k2_scratch) cudaFreeAsync(ctx->k2_scratch, st);
    ctx->k2_scratch = nullptr;
    ctx->k2_scratch_bytes = 0;
    KMALLOC(ctx, ctx->k2_scratch, need, st);
    ctx->k2_scratch_bytes = need;
  }
  uint8_t *scr = reinterpret_cast<uint8_t *>(ctx->k2_scratch);
  uint2 *pairs = reinterpret_cast<uint2 *>(scr);
  lst_m = reinterpret_cast<uint64_t *>(scr + 8 * npairs);
  lst_p = reinterpret_cast<uint32_t *>(scr + 8 * npairs + 8 * (size_t)N);
  uint32_t limit = BL_LIMIT;  // KARETO_K2_TABLE_LIMIT (tests) lowers it to exercise the fallback
  if (const char *e = getenv("KARETO_K2_TABLE_LIMIT")) {
    const long v = atol(e);
    if (v >= 0 && v < (long)limit) limit = (uint32_t)v;
  }
  const size_t smem = sizeof(BLTable) * BL_WARPS;
  hm.mark(st, "bounds + allocs");
  {
    Pass ps(ctx, "K2_bucket_link", 1, 1);
    cudaFuncSetAttribute(k_bucket_link, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bucket_link<<<sms, BL_WARPS * 32, smem, st>>>(k32s.p, v64s.p, bstart.p, cstart.p, cbucket.p, ctr.p, cursor.p,
                                                     pairs, rec_m, rec_p, lst_m, lst_p, rec_n.p, ovf_dev, limit, sl, cstride);
  }
  hm.mark(st, "link");
  {
    Pass ps(ctx, "K2_bucket_fixup", 1, 1);
    cudaFuncSetAttribute(k_bucket_fixup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bucket_fixup<<<sms, BL_WARPS * 32, smem, st>>>(bstart.p, cstart.p, ctr.p + 1, cursor.p, pairs, rec_m, rec_p,
                                                      lst_m, lst_p, rec_n.p, ovf_dev, limit, sl, cstride);
  }
  k32.release(); v64.release();
  {
    Pass ps(ctx, "K2_bucket_assemble", 1, 1);
    const unsigned g = (unsigned)(nbk < (uint64_t)(4 * sms) ? nbk : 4 * sms);
    cudaFuncSetAttribute(k_bucket_assemble<PBT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << PBT);
    k_bucket_assemble<PBT><<<g, 1024, 4 << PBT, st>>>(pairs, N, prev, sl);
  }
  hm.mark(st, "fixup + assemble");
  return KARETO_OK;
}

kareto_status link_prev(kareto_ctx *ctx, const uint64_t *hash, uint64_t N, uint32_t *prev, SortedHashes *keep,
                        SortedHashes *prep, unsigned *bucket_ovf) {
  if (N == 0) return KARETO_OK;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  DBuf<uint8_t> tmp;
  DBuf<uint32_t> k32, k32s;
  DBuf<uint64_t> v64, v64s;
  KTRY(k32s.alloc(ctx, N)); KTRY(v64s.alloc(ctx, N));
  if (prep && prep->key.p) {  // written by K1
    k32 = std::move(prep->key);
    v64 = std::move(prep->val);
  } else {
    KTRY(k32.alloc(ctx, N)); KTRY(v64.alloc(ctx, N));
    Pass ps(ctx, "K2_sort_prep", 1, 1);
    k_sort_prep<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(hash, N, k32.p, v64.p);
  }
  // whole-trace loads: 16-bit buckets + the warp bucket link; its table-overflow flag goes to
  // *bucket_ovf, which kareto_load_trace reads at its next host synchronisation (re-running the
  // load with the full sort below if it is set)
  if (!keep && bucket_ovf) return bucket_link(ctx, k32, v64, k32s, v64s, N, prev, tmp, bucket_ovf);
  {
    Pass ps(ctx, "K2_sort_hashes", 0, 1);
    cub::DoubleBuffer<uint32_t> dk(k32.p, k32s.p);
    cub::DoubleBuffer<uint64_t> dv(v64.p, v64s.p);
    KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
      return K2Sort::Dispatch(t, b, dk, dv, (uint32_t)N, 0, 32, true, st);
    }));
    if (dk.Current() != k32s.p) {  // the result lives in whichever buffer the passes ended in
      std::swap(k32.p, k32s.p);
      std::swap(v64.p, v64s.p);
    }
  }
  k32.release(); v64.release();
  uint8_t *qf = nullptr, *nx = nullptr;
  if (keep) {
    KTRY(keep->qf.alloc(ctx, N)); KTRY(keep->nx.alloc(ctx, N)); KTRY(keep->nx.zero());
    qf = keep->qf.p;
    nx = keep->nx.p;
  }
  {
    DBuf<uint2> pairs, ovf;
    DBuf<uint32_t> n_ovf;
    DBuf<unsigned> cursor;
    constexpr int PBT = 15;
    const uint64_t nbk_t = (N + (1u << PBT) - 1) >> PBT;
    const bool tiled = nbk_t <= (uint64_t)LT_MAX_BUCKETS;
    const int pbits = tiled ? PBT : PB;
    const uint64_t nbk = (N + (1ull << pbits) - 1) >> pbits;
    KTRY(pairs.alloc(ctx, N)); KTRY(ovf.alloc(ctx, N)); KTRY(n_ovf.alloc(ctx, 1)); KTRY(n_ovf.zero());
    KTRY(cursor.alloc(ctx, nbk)); KTRY(cursor.zero());
    {
      Pass ps(ctx, "K2_link_prev", 1, 1);
      if (tiled) {
        const size_t smem = 8 * (size_t)LT_TILE + 8 * (size_t)nbk;
        cudaFuncSetAttribute(k_link_tile<PBT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const uint64_t ntile = (N + LT_TILE - 1) / LT_TILE;
        k_link_tile<PBT><<<(unsigned)(ntile < (uint64_t)(2 * sms) ? ntile : 2 * sms), LT_THREADS, smem, st>>>(
            k32s.p, v64s.p, N, (int)nbk, cursor.p, pairs.p, ovf.p, n_ovf.p, qf, nx);
      } else {
        k_link_prev<<<grid_for((N + LINK_U - 1) / LINK_U, 256, 8 * sms), 256, 0, st>>>(
            k32s.p, v64s.p, N, cursor.p, pairs.p, ovf.p, n_ovf.p, qf, nx);
      }
    }
    {
      Pass ps(ctx, "K2_link_overflow", 1, 1);
      k_link_overflow<<<2 * sms, OVF_THREADS, 0, st>>>(k32s.p, v64s.p, ovf.p, n_ovf.p, pairs.p, qf, nx);
    }
    if (getenv("KARETO_DEBUG")) {
      uint32_t h = 0;
      cudaMemcpyAsync(&h, n_ovf.p, 4, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      fprintf(stderr, "[kareto] K2 link overflow elements: %u of %llu\n", h, (unsigned long long)N);
    }
    {
      Pass ps(ctx, "K2_bucket_assemble", 1, 1);
      const unsigned g = (unsigned)(nbk < (uint64_t)(4 * sms) ? nbk : 4 * sms);
      if (tiled) {
        cudaFuncSetAttribute(k_bucket_assemble<PBT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << PBT);
        k_bucket_assemble<PBT><<<g, 1024, 4 << PBT, st>>>(pairs.p, N, prev, 0u);
      } else {
        k_bucket_assemble<PB><<<g, 1024, 4 << PB, st>>>(pairs.p, N, prev, 0u);
      }
    }
  }
  if (keep) {
    keep->key = std::move(k32s);
    keep->val = std::move(v64s);
  }
  return KARETO_OK;
}

static kareto_status load(kareto_ctx *ctx, const kareto_trace_desc *d, kareto_trace **out) {
  kareto_trace *tr = new kareto_trace();
  tr->ctx = ctx;
  tr->stream = ctx->stream;
  struct Guard {
    kareto_trace *&t;
    bool keep = false;
    ~Guard() { if (!keep) kareto_trace_free(t); }
  } guard{tr};
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;

  // ---- a1: sort requests, per-request metadata, block offsets
  HostMarks hm("load");
  Ingest in;
  KTRY(ingest(ctx, d, tr, in));
  hm.mark(st, "a1 ingest");
  const int64_t R = tr->R;
  const uint64_t N = (uint64_t)tr->N;
  LoadStats &hs = in.hs;
  tr->pos_hi = tr->N;
  tr->req_hi = R;

  const uint64_t Na = N > 0 ? N : 1;
  KMALLOC(ctx, tr->hash, 8 * Na, st);
  KMALLOC(ctx, tr->req, 4 * Na, st);
  KMALLOC(ctx, tr->prev, 4 * Na, st);
  KMALLOC(ctx, tr->delta, 4 * Na, st);
  KMALLOC(ctx, tr->depth, 4 * Na, st);

  // ---- a2: K1 chained hashes (TOKENS) / copy (HASHES) into touch order
  SortedHashes prep;  // K2's sort input, written by K1 in TOKENS mode
  {
    DBuf<uint32_t> h_tok;
    DBuf<uint64_t> h_bh;
    const uint32_t *tok_base;
    const uint64_t *bh_base;
    KTRY(upload_payload(ctx, d, 0, in.total, h_tok, h_bh, &tok_base, &bh_base));
    KTRY(chain_hash(ctx, d, tr, in, tok_base, bh_base, in.total, 0, R, tr->hash, tr->req, &prep));
  }
  hm.mark(st, "a2 K1");

  // ---- a3: K2 prev / delta / chain check
  // per run (k_access_flags + k_run_delta) unless KARETO_K2_ACCESS_INFO asks for the per-access
  // k_access_info (kept for comparison; both are parity-tested)
  const bool per_run = getenv("KARETO_K2_ACCESS_INFO") == nullptr;
  RunList rl;
  DBuf<uint32_t> first_cnt, reuse_cnt;
  DBuf<uint8_t> run_flag;
  DBuf<unsigned> k2ovf;
  KTRY(run_flag.alloc(ctx, N > 0 ? N : 1));
  KTRY(first_cnt.alloc(ctx, R)); KTRY(reuse_cnt.alloc(ctx, R));
  KTRY(first_cnt.zero()); KTRY(reuse_cnt.zero());
  if (N > 0) {
    const bool buckets = !ctx->k2_full && getenv("KARETO_K2_FULLSORT") == nullptr;
    if (buckets) { KTRY(k2ovf.alloc(ctx, 1)); KTRY(k2ovf.zero()); }
    KTRY(link_prev(ctx, tr->hash, N, tr->prev, nullptr, &prep, buckets ? k2ovf.p : nullptr));
    hm.mark(st, "a3 K2 link");
    if (per_run) {
      Pass ps(ctx, "K2_access_flags", 1, 1);
      k_access_flags<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->prev, tr->req, tr->s, tr->delta, run_flag.p,
                                                                in.stats.p);
    } else {
      Pass ps(ctx, "K2_access_info", 1, 1);
      k_access_info<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, tr->prev, tr->req, tr->s, tr->arr, tr->hash,
                                                               tr->delta, first_cnt.p, reuse_cnt.p, run_flag.p,
                                                               in.stats.p);
    }
    // K3's run list (heads compacted on the device; M comes back with the groups' round trip)
    KTRY(run_list_start(ctx, N, run_flag.p, rl));
  }

  hm.mark(st, "a3 K2 access_info");
  // ---- a3: groups (top-K prefix subtrees by reuse, residual K)
  {
    DBuf<uint8_t> tmp;
    const int K = tr->K;
    DBuf<uint64_t> rkey, rkey_s, rankkey, rankkey_s;
    DBuf<uint32_t> rval, rval_c, rval_s, head, run_incl, rankidx, ranked, rank, nruns;
    DBuf<uint8_t> rflag;
    DBuf<int> m_dev;
    DBuf<unsigned long long> run_reuse, gtab;
    KTRY(rkey.alloc(ctx, R)); KTRY(rkey_s.alloc(ctx, R)); KTRY(rval.alloc(ctx, R)); KTRY(rval_c.alloc(ctx, R));
    KTRY(rval_s.alloc(ctx, R)); KTRY(head.alloc(ctx, R)); KTRY(run_incl.alloc(ctx, R)); KTRY(rflag.alloc(ctx, R));
    KTRY(m_dev.alloc(ctx, 1)); KTRY(run_reuse.alloc(ctx, R)); KTRY(run_reuse.zero()); KTRY(nruns.alloc(ctx, 1));
    KTRY(nruns.zero());
    KTRY(rankkey.alloc(ctx, R)); KTRY(rankkey_s.alloc(ctx, R)); KTRY(rankidx.alloc(ctx, R)); KTRY(ranked.alloc(ctx, R));
    KTRY(rank.alloc(ctx, R)); KTRY(gtab.alloc(ctx, 2 * (K + 1))); KTRY(gtab.zero());
    DBuf<uint64_t> rkey_c;
    KTRY(rkey_c.alloc(ctx, R));
    {
    Pass ps(ctx, "K2g_select", 1, 1);
    k_root_keys<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(R, tr->s, tr->hash, 0, rkey.p, rval.p, rflag.p);
    KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceSelect::Flagged(t, b, rkey.p, rflag.p, rkey_c.p, m_dev.p, (int)R, st);
    }));
    KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceSelect::Flagged(t, b, rval.p, rflag.p, rval_c.p, m_dev.p, (int)R, st);
    }));
    }
    int m = 0, M = 0;
    unsigned k2o = 0;
    KCUDA(ctx, cudaMemcpyAsync(&m, m_dev.p, 4, cudaMemcpyDeviceToHost, st));
    if (N > 0) KCUDA(ctx, cudaMemcpyAsync(&M, rl.m_dev.p, 4, cudaMemcpyDeviceToHost, st));
    if (k2ovf.p) KCUDA(ctx, cudaMemcpyAsync(&k2o, k2ovf.p, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    if (k2o) {  // a bucket exceeded the link table: prev is valid but not exact -- redo with the full sort
      if (getenv("KARETO_DEBUG")) fprintf(stderr, "[kareto] K2 bucket link: table overflow, full-sort re-run\n");
      return KARETO_RETRY_FULL_SORT;
    }
    if (N > 0) {  // the run list, and per run the reuse interval and the chain checks
      KTRY(run_list_finish(ctx, N, tr->prev, tr->req, 0, tr->s, 0, M, rl));
      if (per_run) {
        Pass ps(ctx, "K2_run_delta", 1, 2);
        if (M > 0)
          k_run_delta<<<grid_for(M, 256, 16 * sms), 256, 0, st>>>(rl.m_dev.p, rl.run_start.p, rl.run_req.p,
                                                                  rl.run_len.p, rl.run_p0.p, tr->prev, tr->req, tr->s,
                                                                  tr->arr, tr->hash, tr->delta, reuse_cnt.p,
                                                                  in.stats.p);
        k_first_from_reuse<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(R, tr->s, reuse_cnt.p, first_cnt.p);
      }
    }
    k_fill_u16<<<grid_for(R, 256, 4 * sms), 256, 0, st>>>(tr->grp, R, (uint16_t)K);
    if (m > 0) {
      {
      Pass ps(ctx, "K2g_sort_roots", 0, 1);
      KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, rkey_c.p, rkey_s.p, rval_c.p, rval_s.p, m, 0, 64, st);
      }));
      }
      Pass ps(ctx, "K2g_rank", 1, 6);
      k_run_heads<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(rkey_s.p, m_dev.p, head.p);
      KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceScan::InclusiveSum(t, b, head.p, run_incl.p, m, st);
      }));
      k_run_reuse<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(rval_s.p, run_incl.p, m_dev.p, reuse_cnt.p, run_reuse.p,
                                                             nruns.p);
      k_rank_keys<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(run_reuse.p, nruns.p, rankkey.p, rankidx.p, (uint32_t)m);
      KTRY(cub_call(ctx, tmp, [&](void *t, size_t &b) {
        // reuse < 2^32: the low 32 bits of ~reuse order runs the same way (4 passes instead of 8)
        return cub::DeviceRadixSort::SortPairs(t, b, rankkey.p, rankkey_s.p, rankidx.p, ranked.p, m, 0, 32, st);
      }));
      k_rank_of_run<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(ranked.p, nruns.p, rank.p);
      k_assign_groups<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(rval_s.p, run_incl.p, m_dev.p, rank.p, K, tr->grp);
    }
    Pass ps2(ctx, "K2g_tables", 1, 1);
    k_group_tables<<<grid_for(R, 256, 4 * sms), 256, 16 * (K + 1), st>>>(R, 0, tr->grp, first_cnt.p, reuse_cnt.p,
                                                                          gtab.p, K + 1);
    std::vector<unsigned long long> h(2 * (K + 1));
    KCUDA(ctx, cudaMemcpyAsync(h.data(), gtab.p, 16 * (K + 1), cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaMemcpyAsync(&hs, in.stats.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    tr->U_g.resize(K + 1);
    tr->reuse_g.resize(K + 1);
    int64_t U = 0;
    for (int g = 0; g <= K; g++) {
      tr->U_g[g] = (int64_t)h[2 * g];
      tr->reuse_g[g] = (int64_t)h[2 * g + 1];
      U += tr->U_g[g];
    }
    tr->U = U;
  }
  if (hs.flags & F_CHAIN) return fail(ctx, KARETO_E_CHAIN, "block hashes are not chain-consistent (R7)");
  if (hs.flags & F_DELTA) return fail(ctx, KARETO_E_OVERFLOW, "a reuse interval >= 2^32-1 ms");

  hm.mark(st, "a3 K2 groups");
  // ---- a4: K3 LRU stack depths
  if (N > 0) {
    if (N >= (1ull << 31)) return fail(ctx, KARETO_E_OVERFLOW, "stack depth pass supports < 2^31 accesses");
    // the runs are kept and per-access depths deferred to their first reader (ensure_depth)
    KTRY(stack_depth_runs(ctx, N, N, tr->s, 0, 0, rl, nullptr, &tr->n_runs, &tr->runs));
    tr->depth_ready = false;
  }
  KTRY(sync(ctx, "load_trace"));
  hm.mark(st, "a4 K3");
  if (getenv("KARETO_POOLSTAT")) {
    size_t rsv = 0, used = 0, hi = 0;
    cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &rsv);
    cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemCurrent, &used);
    cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemHigh, &hi);
    fprintf(stderr, "[pool] reserved %.2f GB (high %.2f) used %.2f GB\n", rsv / 1e9, hi / 1e9, used / 1e9);
  }
  guard.keep = true;
  *out = tr;
  return KARETO_OK;
}

}  // namespace kareto

extern "C" kareto_status kareto_load_trace(kareto_ctx *ctx, const kareto_trace_desc *desc, kareto_trace **out) {
  if (!ctx || !desc || !out) return KARETO_E_INVALID;
  *out = nullptr;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::load(ctx, desc, out);
  if (s == kareto::KARETO_RETRY_FULL_SORT) {  // rare: some K2 bucket overflowed the warp tables
    cudaStreamSynchronize(ctx->stream);
    ctx->k2_full = true;
    s = kareto::load(ctx, desc, out);
    ctx->k2_full = false;
  }
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

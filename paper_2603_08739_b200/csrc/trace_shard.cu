// trace_shard.cu -- row f4: time-sharded trace passes, kareto_load_trace_sharded.
//
// Rank k of W owns the sorted requests [r_k, r_{k+1}) whose blocks occupy the positions
// [P0, P1) ~ [kN/W, (k+1)N/W) of the touch order, and runs K1 (hash), K2 (prev, delta, chain
// check, groups), K3 (LRU depth) on them only; K4 histograms are summed across ranks at
// evaluation time (eval.cu).  The result is identical, access by access, to the whole-trace
// load (kareto_load_trace): same prev (global positions), delta, depth, groups, U.
//
// What crosses shard boundaries, and how:
//   * prev of the first access of a block inside the shard (a "Q" record) is the last access of
//     that block in an earlier shard (its "P" record).  Every rank sends, for each distinct block
//     of its shard, a Q record (first access) and a P record (last access) to the OWNER rank of
//     the block's hash (hash partitioned: all-to-all-v, 24 B per record, each source's records
//     in key order).  The owner (one CTA per key bucket, no sort: each source chunk is binary
//     searched) answers each Q with the P of the latest earlier shard holding the block (or
//     "globally first"), checking chain consistency across the boundary (R7), and each P with
//     the next shard holding the block; answers return by a second all-to-all-v.
//   * depth needs the LRU stack at the shard boundary P0: B_k = {last access before P0 of every
//     block seen before P0}.  A P record at shard j whose block next appears in shard n (W if
//     never) belongs to B_k exactly for j < k <= n, so shard j sends rank k > j a bitmap of its
//     positions with n >= k (ballot-packed, 1 bit per position; third all-to-all-v) and rank k
//     ORs them into B_k over [0, P0).  Rank k then solves its shard as a standalone trace
//     prefixed by B_k in position order (virtual accesses of distinct blocks): a previous
//     position p < P0 maps to its rank in B_k (prefix popcounts), p >= P0 to |B_k| + p - P0,
//     and K3 runs unchanged on the compressed coordinates.  Exact: the distinct blocks touched
//     in [p, s_r) of the real trace are those of B_k at or after p plus those touched in
//     [P0, s_r), as in the virtual trace.
//   * groups (R23) need the global reuse of every prefix subtree: per-rank (root hash, reuse)
//     tables are all-gathered and reduced identically on every rank.
//   * U, U_g, reuse_g and the error flags: one allreduce.
#include <cub/cub.cuh>

#include "trace_load.cuh"

namespace kareto {

struct XRec {       // exchange record, 24 B
  uint64_t m;       // fmix64(h ^ kSortMixC): a bijection of the block hash; key32 = m >> 32
  uint64_t parent;  // hash of the parent block (chain position k - 1); 0 for roots
  uint32_t pos;     // global position of the access
  uint32_t info;    // bit 31: P (last access in its shard) / 0: Q (first); bits 24..30: source
                    // rank; bits 0..23: chain position k
};
constexpr uint32_t kRecP = 0x80000000u;
constexpr int kMaxShardWorld = 128;
constexpr uint32_t kChainPosMask = 0x00FFFFFFu;

__host__ __device__ __forceinline__ uint32_t owner_of(uint32_t key32, int W) {
  return (uint32_t)(((uint64_t)key32 * (uint64_t)W) >> 32);
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

// r_k = first request with s[r] >= k N / W (k = 0..W-1), r_W = R (host and device)
__host__ __device__ inline uint32_t slice_bound(const uint32_t *s, int64_t R, uint64_t N, int W, int k) {
  if (k >= W) return (uint32_t)R;
  uint64_t target = (N * (uint64_t)k) / (uint64_t)W;
  int64_t lo = 0, hi = R;
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if ((uint64_t)s[m] >= target) hi = m; else lo = m + 1;
  }
  return (uint32_t)lo;
}
__global__ void k_slice_bounds(const uint32_t *__restrict__ s, int64_t R, uint64_t N, int W, uint32_t *__restrict__ rb) {
  int k = threadIdx.x;
  if (k <= W) rb[k] = slice_bound(s, R, N, W, k);
}

// Records per fingerprint-sorted element: Q if it is the first access of its block in the shard,
// P if the last (flags from the link kernels: qf, nx).  fl bit 0 = Q, bit 1 = P; cnt = popcount.
__global__ void k_rec_flags(const uint8_t *__restrict__ qf, const uint8_t *__restrict__ nx, uint64_t n,
                            uint8_t *__restrict__ fl, uint32_t *__restrict__ cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = qf[i] ? 1u : 0u, p = nx[i] ? 0u : 1u;
    fl[i] = (uint8_t)(q | (p << 1));
    cnt[i] = q + p;
  }
}

__global__ void k_rec_emit(const uint32_t *__restrict__ ks, const uint64_t *__restrict__ vs, uint64_t n,
                           const uint8_t *__restrict__ fl, const uint32_t *__restrict__ off, const uint32_t *__restrict__ req,
                           const uint32_t *__restrict__ s, const uint64_t *__restrict__ hash, uint32_t P0, int rank,
                           XRec *__restrict__ rec) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = vs[i];
    const uint32_t j = (uint32_t)v;
    const uint8_t f = fl[i];
    if (!f) continue;
    const bool q = f & 1, p = f & 2;
    XRec x;
    x.m = ((uint64_t)ks[i] << 32) | (v >> 32);
    x.pos = P0 + j;
    const uint32_t k = s[req[j] + 1] - 1 - x.pos;
    x.parent = k > 0 ? hash[j + 1] : 0ull;
    x.info = ((uint32_t)rank << 24) | (k & kChainPosMask);
    uint32_t o = off[i];
    if (q) rec[o++] = x;
    if (p) { x.info |= kRecP; rec[o] = x; }
  }
}

// send boundaries: first record of each owner (records are in key32 order)
__global__ void k_owner_bounds(const XRec *__restrict__ rec, uint32_t n, int W, uint32_t *__restrict__ ob) {
  int o = threadIdx.x;
  if (o > W) return;
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t m = (lo + hi) >> 1;
    if (owner_of((uint32_t)(rec[m].m >> 32), W) >= (uint32_t)o) hi = m; else lo = m + 1;
  }
  ob[o] = lo;
}

// Owner (one CTA per key bucket).  The records of source rank c arrive as chunk c, sorted by
// key (then position); a bucket's records of chunk c are a contiguous subrange found by binary
// search, and every record of one block lies in one bucket.  Q record of chunk c: answer with
// the P record of the same block in the LATEST chunk c' < c holding it (or kNone = globally
// first access), checking chain consistency (R7) across the boundary; P record: answer with
// the EARLIEST later chunk holding the block (W if none).  No sort: each chunk is searched.
constexpr int OWN_THREADS = 256;

// A bucket's records are staged in shared memory (chunk after chunk) when they fit; the
// searches then run on shared memory.  Larger buckets (never seen with uniform keys; possible
// only for adversarial hashes) search global memory.
constexpr int OWN_STAGE = 1536;  // records (36 KB)
template <bool SMEM>
__device__ __forceinline__ void owner_bucket(const XRec *__restrict__ g, const XRec *__restrict__ sm,
                                             const uint32_t *lo, const uint32_t *hi, const uint32_t *pre, int W,
                                             uint32_t *__restrict__ reply, unsigned &bad) {
  // record t of the bucket (chunk c): global index lo[c] + (t - pre[c]); staged index t
  const uint32_t tot = pre[W];
  auto rec_at = [&](int c, uint32_t t) -> const XRec & { return SMEM ? sm[t] : g[lo[c] + (t - pre[c])]; };
  auto key_at = [&](int c, uint32_t t) -> uint32_t { return (uint32_t)(rec_at(c, t).m >> 32); };
  auto lb = [&](int c, uint32_t key) -> uint32_t {  // first staged index of chunk c with key >= key
    uint32_t a = pre[c], b = pre[c + 1];
    while (a < b) {
      uint32_t m = (a + b) >> 1;
      if (key_at(c, m) < key) a = m + 1; else b = m;
    }
    return a;
  };
  for (uint32_t t = threadIdx.x; t < tot; t += blockDim.x) {
    int c = 0;
    while (pre[c + 1] <= t) c++;
    const XRec x = rec_at(c, t);
    const uint32_t key = (uint32_t)(x.m >> 32);
    uint32_t ans;
    if (!(x.info & kRecP)) {
      ans = kNone;
      for (int c2 = c - 1; c2 >= 0 && ans == kNone; c2--) {
        for (uint32_t u = lb(c2, key); u < pre[c2 + 1] && key_at(c2, u) == key; u++) {
          const XRec &y = rec_at(c2, u);
          if (y.m != x.m || !(y.info & kRecP)) continue;
          ans = y.pos;
          const uint32_t kq = x.info & kChainPosMask, kp = y.info & kChainPosMask;
          if (kq != kp || (kq > 0 && y.parent != x.parent)) bad++;
          break;
        }
      }
    } else {
      ans = (uint32_t)W;
      for (int c2 = c + 1; c2 < W && ans == (uint32_t)W; c2++)
        for (uint32_t u = lb(c2, key); u < pre[c2 + 1] && key_at(c2, u) == key; u++)
          if (rec_at(c2, u).m == x.m) { ans = (uint32_t)c2; break; }
    }
    reply[lo[c] + (t - pre[c])] = ans;
  }
}

// bucket of an owned key: (key - klo) >> shift (buckets of 2^shift consecutive keys)
__device__ __forceinline__ uint32_t bucket_of(uint32_t klo, int shift, uint32_t key) { return (key - klo) >> shift; }
// bnd[c * (B + 1) + b] = first record of chunk c in bucket >= b (one pass over the records:
// each record writes the boundaries between its predecessor's bucket and its own)
__global__ void k_bucket_bounds(const XRec *__restrict__ in, const uint64_t *__restrict__ co, int W, uint32_t klo,
                                int shift, uint32_t B, uint32_t n, uint32_t *__restrict__ bnd) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int c = 0;
    while (co[c + 1] <= i) c++;
    const bool first = i == (uint32_t)co[c], last = i + 1 == (uint32_t)co[c + 1];
    const uint32_t b = bucket_of(klo, shift, (uint32_t)(in[i].m >> 32));
    const int64_t bp = first ? -1 : (int64_t)bucket_of(klo, shift, (uint32_t)(in[i - 1].m >> 32));
    uint32_t *row = bnd + (size_t)c * (B + 1);
    for (int64_t x = bp + 1; x <= (int64_t)b; x++) row[x] = i;
    if (last)
      for (uint32_t x = b + 1; x <= B; x++) row[x] = i + 1;
  }
}
// chunks without records: every boundary at the chunk start
__global__ void k_bucket_bounds_empty(const uint64_t *__restrict__ co, int W, uint32_t B, uint32_t *__restrict__ bnd) {
  for (int c = 0; c < W; c++) {
    if (co[c + 1] != co[c]) continue;
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= B; x += gridDim.x * blockDim.x)
      bnd[(size_t)c * (B + 1) + x] = (uint32_t)co[c];
  }
}

__global__ void __launch_bounds__(OWN_THREADS) k_owner(const XRec *__restrict__ in, const uint32_t *__restrict__ bnd,
                                                       int W, uint32_t B, uint32_t *__restrict__ reply,
                                                       unsigned long long *__restrict__ flags) {
  __shared__ uint32_t lo[kMaxShardWorld], hi[kMaxShardWorld], pre[kMaxShardWorld + 1];
  __shared__ XRec stage[OWN_STAGE];
  unsigned bad = 0;
  for (uint32_t b = blockIdx.x; b < B; b += gridDim.x) {
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
      lo[c] = bnd[(size_t)c * (B + 1) + b];
      hi[c] = bnd[(size_t)c * (B + 1) + b + 1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      pre[0] = 0;
      for (int c = 0; c < W; c++) pre[c + 1] = pre[c] + (hi[c] - lo[c]);
    }
    __syncthreads();
    const uint32_t tot = pre[W];
    if (tot <= (uint32_t)OWN_STAGE) {
      for (uint32_t t = threadIdx.x; t < tot; t += blockDim.x) {
        int c = 0;
        while (pre[c + 1] <= t) c++;
        stage[t] = in[lo[c] + (t - pre[c])];
      }
      __syncthreads();
      owner_bucket<true>(in, stage, lo, hi, pre, W, reply, bad);
    } else {
      owner_bucket<false>(in, stage, lo, hi, pre, W, reply, bad);
    }
    __syncthreads();
  }
  if (bad) atomicAdd(&flags[0], (unsigned long long)bad);
}

// prev in global positions: in-shard links + the owners' answers for the Q records
__global__ void k_prev_global(const uint32_t *__restrict__ prev_loc, uint64_t n, uint32_t P0, uint32_t *__restrict__ prev) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t p = prev_loc[i];
    prev[i] = p == kNone ? kNone : P0 + p;
  }
}
// Q answers -> prev; P answers -> nxs[local position] = the next shard holding the block
__global__ void k_apply_replies(const XRec *__restrict__ rec, const uint32_t *__restrict__ reply, uint32_t n,
                                uint32_t P0, uint32_t *__restrict__ prev, uint8_t *__restrict__ nxs) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const XRec x = rec[i];
    if (!(x.info & kRecP)) prev[x.pos - P0] = reply[i];
    else nxs[x.pos - P0] = (uint8_t)reply[i];
  }
}

// Boundary-set bitmaps this shard contributes to every later rank k: bit p set iff p is the last
// access of its block in this shard and the block next appears in shard k or later (or never),
// i.e. p in B_k.  Words are aligned to global positions (word w covers [32w, 32w+32)); one
// read of each position's next-shard byte, one ballot per later rank; out + (k - me - 1) * nwords
// is rank k's bitmap.
__global__ void k_bset_words(const uint8_t *__restrict__ nxs, uint32_t P0, uint32_t P1, uint32_t w0, uint32_t nwords,
                             int me, int W, uint32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < (uint64_t)nwords * 32;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = (w0 << 5) + (uint32_t)t;  // one position per thread, a warp per word
    const int nx = (p >= P0 && p < P1) ? nxs[p - P0] : 0;
    for (int k = me + 1; k < W; k++) {
      const unsigned w = __ballot_sync(0xFFFFFFFFu, nx >= k);
      if (lane == 0) out[(size_t)(k - me - 1) * nwords + (t >> 5)] = w;
    }
  }
}
// OR a received word segment into the bitmap (neighbouring shards share a boundary word)
__global__ void k_or_words(const uint32_t *__restrict__ seg, uint32_t w0, uint32_t n, uint32_t nbits_words,
                           uint32_t *__restrict__ bits) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (w0 + i < nbits_words && seg[i]) atomicOr(&bits[w0 + i], seg[i]);
}

__global__ void k_popc(const uint32_t *__restrict__ bits, uint64_t nw, uint32_t *__restrict__ pc) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x)
    pc[i] = __popc(bits[i]);
}

__device__ __forceinline__ void warp_count_add(uint32_t *arr, uint32_t key, bool pred) {
  const unsigned active = __activemask();
  const unsigned pm = __ballot_sync(active, pred);
  if (!pred) return;
  const unsigned same = __match_any_sync(pm, key);
  if ((__ffs(same) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&arr[key], (uint32_t)__popc(same));
}

// delta, chain check (in-shard links; cross-shard links were checked by the owners), K3 run
// heads, per-request first/reuse counts, compressed previous positions for K3
__global__ void k_access_info_shard(uint64_t n, uint32_t P0, uint32_t r0, const uint32_t *__restrict__ prev,
                                    const uint32_t *__restrict__ req, const uint32_t *__restrict__ s, int64_t R,
                                    const int64_t *__restrict__ arr, const uint64_t *__restrict__ hash,
                                    const uint32_t *__restrict__ bits, const uint32_t *__restrict__ pre, uint32_t Bsize,
                                    uint32_t *__restrict__ delta, uint32_t *__restrict__ prev_c,
                                    uint32_t *__restrict__ first_cnt, uint32_t *__restrict__ reuse_cnt,
                                    uint8_t *__restrict__ run_flag, unsigned long long *__restrict__ flags) {
  unsigned fl_chain = 0, fl_delta = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = prev[i], r = req[i], j = P0 + (uint32_t)i;
    uint32_t dl = kNone, pc = kNone;
    if (p != kNone) {
      uint32_t rp;
      if (p >= P0) {
        rp = req[p - P0];
        pc = Bsize + (p - P0);
        const uint32_t kj = s[r + 1] - 1 - j, kp = s[rp + 1] - 1 - p;
        if (kj != kp) fl_chain++;
        else if (kj > 0 && prev[i + 1] != p + 1 && hash[i + 1] != hash[p - P0 + 1]) fl_chain++;
      } else {
        int64_t lo = 0, hi = R;  // last request with s[r] <= p
        while (lo < hi) {
          int64_t m = (lo + hi + 1) >> 1;
          if (s[m] <= p) lo = m; else hi = m - 1;
        }
        rp = (uint32_t)lo;
        const uint32_t w = bits[p >> 5];
        pc = pre[p >> 5] + __popc(w & ((1u << (p & 31)) - 1u));
      }
      int64_t d = arr[r] - arr[rp];
      if (d < 0 || d >= (int64_t)kNone) fl_delta++; else dl = (uint32_t)d;
    }
    delta[i] = dl;
    prev_c[i] = pc;
    uint8_t head = 0;
    if (p != kNone) {
      const uint32_t pm = i > 0 ? prev[i - 1] : kNone;
      head = (j == s[r] || pm == kNone || p != pm + 1) ? 1 : 0;
    }
    run_flag[i] = head;
    warp_count_add(first_cnt, r - r0, p == kNone);
    warp_count_add(reuse_cnt, r - r0, p != kNone);
  }
  if (fl_chain) atomicAdd(&flags[0], (unsigned long long)fl_chain);
  if (fl_delta) atomicAdd(&flags[1], (unsigned long long)fl_delta);
}

// groups: reuse of each root over the shard's requests
__global__ void k_root_reuse(const uint32_t *__restrict__ rval, const int *__restrict__ m_ptr,
                             const uint32_t *__restrict__ reuse_cnt, unsigned long long *__restrict__ v) {
  int m = *m_ptr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) v[i] = reuse_cnt[rval[i]];
}
__global__ void k_concat_tables(const uint64_t *__restrict__ gk, const unsigned long long *__restrict__ gv,
                                const uint64_t *__restrict__ cnt_off, int W, uint64_t stride, uint64_t *__restrict__ k,
                                unsigned long long *__restrict__ v) {
  for (int r = 0; r < W; r++) {
    const uint64_t c = cnt_off[r + 1] - cnt_off[r];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < c; i += (uint64_t)gridDim.x * blockDim.x) {
      k[cnt_off[r] + i] = gk[r * stride + i];
      v[cnt_off[r] + i] = gv[r * stride + i];
    }
  }
}
__global__ void k_rank_keys32(const unsigned long long *__restrict__ tot, uint32_t n, uint32_t *__restrict__ key,
                              uint32_t *__restrict__ idx) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    key[i] = ~(uint32_t)tot[i];  // reuse < 2^32; stable sort => (reuse desc, root hash asc)
    idx[i] = i;
  }
}
__global__ void k_top_table(const uint32_t *__restrict__ ranked, const uint64_t *__restrict__ roots, uint32_t ntop,
                            uint64_t *__restrict__ th, uint32_t *__restrict__ trk) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ntop; i += gridDim.x * blockDim.x) {
    th[i] = roots[ranked[i]];
    trk[i] = i;
  }
}
__global__ void k_group_lookup(int64_t n, const uint64_t *__restrict__ rkey, const uint8_t *__restrict__ rflag,
                               const uint64_t *__restrict__ th, const uint32_t *__restrict__ trk, uint32_t ntop,
                               int K, uint16_t *__restrict__ grp) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t g = (uint32_t)K;
    if (rflag[r]) {
      const uint64_t h = rkey[r];
      uint32_t lo = 0, hi = ntop;
      while (lo < hi) {
        uint32_t m = (lo + hi) >> 1;
        if (th[m] < h) lo = m + 1; else hi = m;
      }
      if (lo < ntop && th[lo] == h) g = trk[lo];
    }
    grp[r] = (uint16_t)g;
  }
}

// kernels shared with the whole-trace load (trace_load.cu)
__global__ void k_root_keys(int64_t R, const uint32_t *__restrict__ s, const uint64_t *__restrict__ hash,
                            uint32_t pos_base, uint64_t *__restrict__ key, uint32_t *__restrict__ val,
                            uint8_t *__restrict__ flag);
__global__ void k_group_tables(int64_t R, uint32_t r_base, const uint16_t *__restrict__ grp,
                               const uint32_t *__restrict__ first_cnt, const uint32_t *__restrict__ reuse_cnt,
                               unsigned long long *__restrict__ tab, int G);
__global__ void k_fill_u16(uint16_t *p, int64_t n, uint16_t v);

static std::vector<size_t> offsets_of(const std::vector<uint64_t> &cnt, size_t elem) {
  std::vector<size_t> o(cnt.size() + 1, 0);
  for (size_t i = 0; i < cnt.size(); i++) o[i + 1] = o[i] + (size_t)cnt[i] * elem;
  return o;
}

// groups (R23) over the whole trace from the shards' (root, reuse) tables
static kareto_status shard_groups(kareto_ctx *ctx, kareto_trace *tr, const uint32_t *reuse_cnt) {
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms, W = ctx->world, K = tr->K;
  const int64_t r0 = tr->req_lo, nr = tr->req_hi - tr->req_lo;
  const int64_t nra = nr > 0 ? nr : 1;
  DBuf<uint8_t> tmp, rflag;
  DBuf<uint64_t> rkey, rkey_c, rkey_s, uroots;
  DBuf<uint32_t> rval, rval_c, rval_s;
  DBuf<unsigned long long> rv, usum;
  DBuf<int> m_dev, nu_dev;
  KTRY(rflag.alloc(ctx, nra)); KTRY(rkey.alloc(ctx, nra)); KTRY(rkey_c.alloc(ctx, nra)); KTRY(rkey_s.alloc(ctx, nra));
  KTRY(uroots.alloc(ctx, nra)); KTRY(rval.alloc(ctx, nra)); KTRY(rval_c.alloc(ctx, nra)); KTRY(rval_s.alloc(ctx, nra));
  KTRY(rv.alloc(ctx, nra)); KTRY(usum.alloc(ctx, nra)); KTRY(m_dev.alloc(ctx, 1)); KTRY(nu_dev.alloc(ctx, 1));
  KTRY(m_dev.zero()); KTRY(nu_dev.zero());
  int nu = 0;
  if (nr > 0) {
    k_root_keys<<<grid_for(nr, 256, 4 * sms), 256, 0, st>>>(nr, tr->s + r0, tr->hash, (uint32_t)tr->pos_lo, rkey.p,
                                                            rval.p, rflag.p);
    ctx->own_launches++;
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceSelect::Flagged(t, b, rkey.p, rflag.p, rkey_c.p, m_dev.p, (int)nr, st);
    }));
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceSelect::Flagged(t, b, rval.p, rflag.p, rval_c.p, m_dev.p, (int)nr, st);
    }));
    int m = 0;
    KCUDA(ctx, cudaMemcpyAsync(&m, m_dev.p, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    if (m > 0) {
      KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, rkey_c.p, rkey_s.p, rval_c.p, rval_s.p, m, 0, 64, st);
      }));
      k_root_reuse<<<grid_for(m, 256, 4 * sms), 256, 0, st>>>(rval_s.p, m_dev.p, reuse_cnt, rv.p);
      ctx->own_launches++;
      KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
        return cub::DeviceReduce::ReduceByKey(t, b, rkey_s.p, uroots.p, rv.p, usum.p, nu_dev.p, cub::Sum(), m, st);
      }));
      KCUDA(ctx, cudaMemcpyAsync(&nu, nu_dev.p, 4, cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
    }
  }
  // all-gather the per-shard tables (padded to the largest), concatenate, reduce by root
  uint64_t mine = (uint64_t)nu;
  std::vector<uint64_t> cnt(W);
  KTRY(coll_allgather_host(ctx, &mine, cnt.data(), 8));
  uint64_t stride = 1;
  for (int r = 0; r < W; r++) stride = cnt[r] > stride ? cnt[r] : stride;
  std::vector<uint64_t> co(W + 1, 0);
  for (int r = 0; r < W; r++) co[r + 1] = co[r] + cnt[r];
  const uint64_t M = co[W];
  DBuf<uint64_t> pk, gk, ak, ak_s, roots, dco;
  DBuf<unsigned long long> pv, gv, av, av_s, tot;
  KTRY(pk.alloc(ctx, stride)); KTRY(pv.alloc(ctx, stride));
  KTRY(gk.alloc(ctx, stride * W)); KTRY(gv.alloc(ctx, stride * W));
  if (nu > 0) {
    KCUDA(ctx, cudaMemcpyAsync(pk.p, uroots.p, 8 * (size_t)nu, cudaMemcpyDeviceToDevice, st));
    KCUDA(ctx, cudaMemcpyAsync(pv.p, usum.p, 8 * (size_t)nu, cudaMemcpyDeviceToDevice, st));
  }
  KTRY(coll_allgather(ctx, pk.p, gk.p, 8 * stride));
  KTRY(coll_allgather(ctx, pv.p, gv.p, 8 * stride));
  const uint64_t Ma = M > 0 ? M : 1;
  KTRY(ak.alloc(ctx, Ma)); KTRY(av.alloc(ctx, Ma)); KTRY(ak_s.alloc(ctx, Ma)); KTRY(av_s.alloc(ctx, Ma));
  KTRY(roots.alloc(ctx, Ma)); KTRY(tot.alloc(ctx, Ma)); KTRY(dco.alloc(ctx, W + 1));
  KCUDA(ctx, cudaMemcpyAsync(dco.p, co.data(), 8 * (W + 1), cudaMemcpyHostToDevice, st));
  k_fill_u16<<<grid_for(tr->R, 256, 4 * sms), 256, 0, st>>>(tr->grp, tr->R, (uint16_t)K);  // outside the shard: K
  ctx->own_launches++;
  uint32_t ntop = 0;
  DBuf<uint64_t> th, th_s;
  DBuf<uint32_t> trk, trk_s;
  KTRY(th.alloc(ctx, K > 0 ? K : 1)); KTRY(th_s.alloc(ctx, K > 0 ? K : 1));
  KTRY(trk.alloc(ctx, K > 0 ? K : 1)); KTRY(trk_s.alloc(ctx, K > 0 ? K : 1));
  if (M > 0 && K > 0) {
    k_concat_tables<<<grid_for((int64_t)stride, 256, 4 * sms), 256, 0, st>>>(gk.p, gv.p, dco.p, W, stride, ak.p, av.p);
    ctx->own_launches++;
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, ak.p, ak_s.p, av.p, av_s.p, (int64_t)M, 0, 64, st);
    }));
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceReduce::ReduceByKey(t, b, ak_s.p, roots.p, av_s.p, tot.p, nu_dev.p, cub::Sum(), (int64_t)M, st);
    }));
    int nroot = 0;
    KCUDA(ctx, cudaMemcpyAsync(&nroot, nu_dev.p, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    DBuf<uint32_t> rk, rk_s, ri, ri_s;
    KTRY(rk.alloc(ctx, nroot)); KTRY(rk_s.alloc(ctx, nroot)); KTRY(ri.alloc(ctx, nroot)); KTRY(ri_s.alloc(ctx, nroot));
    k_rank_keys32<<<grid_for(nroot, 256, 4 * sms), 256, 0, st>>>(tot.p, (uint32_t)nroot, rk.p, ri.p);
    ctx->own_launches++;
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, rk.p, rk_s.p, ri.p, ri_s.p, nroot, 0, 32, st);
    }));
    ntop = (uint32_t)(nroot < K ? nroot : K);
    k_top_table<<<grid_for(ntop, 256), 256, 0, st>>>(ri_s.p, roots.p, ntop, th.p, trk.p);
    ctx->own_launches++;
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortPairs(t, b, th.p, th_s.p, trk.p, trk_s.p, (int)ntop, 0, 64, st);
    }));
  }
  if (nr > 0) {
    k_group_lookup<<<grid_for(nr, 256, 4 * sms), 256, 0, st>>>(nr, rkey.p, rflag.p, th_s.p, trk_s.p, ntop, K,
                                                               tr->grp + r0);
    ctx->own_launches++;
  }
  return KARETO_OK;
}

static kareto_status load_sharded(kareto_ctx *ctx, const kareto_trace_desc *d, kareto_trace **out) {
  const int W = ctx->world, me = ctx->rank;
  if (W > kMaxShardWorld) return fail(ctx, KARETO_E_UNSUPPORTED, "time sharding supports world <= %d", kMaxShardWorld);
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

  // ---- a1 (every rank, all requests: R-sized metadata only)
  Ingest in;
  KTRY(ingest(ctx, d, tr, in));
  const int64_t R = tr->R;
  const uint64_t N = (uint64_t)tr->N;
  if (tr->max_blocks > (int32_t)kChainPosMask) return fail(ctx, KARETO_E_UNSUPPORTED, "requests of >= 2^24 blocks");
  if (N >= (1ull << 31)) return fail(ctx, KARETO_E_OVERFLOW, "stack depth pass supports < 2^31 accesses");
  tr->sharded = true;

  // ---- the shard: requests [r0, r1), positions [P0, P1)
  std::vector<uint32_t> rb(W + 1);
  {
    DBuf<uint32_t> drb;
    KTRY(drb.alloc(ctx, W + 1));
    k_slice_bounds<<<1, 256, 0, st>>>(tr->s, R, N, W, drb.p);
    ctx->own_launches++;
    KCUDA(ctx, cudaMemcpyAsync(rb.data(), drb.p, 4 * (W + 1), cudaMemcpyDeviceToHost, st));
  }
  std::vector<uint32_t> sb(W + 1);
  KCUDA(ctx, cudaStreamSynchronize(st));
  for (int k = 0; k <= W; k++) KCUDA(ctx, cudaMemcpyAsync(&sb[k], tr->s + rb[k], 4, cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaStreamSynchronize(st));
  const int64_t r0 = rb[me], r1 = rb[me + 1];
  const uint32_t P0 = sb[me], P1 = sb[me + 1];
  const uint64_t n = P1 - P0, na = n > 0 ? n : 1;
  tr->req_lo = r0; tr->req_hi = r1; tr->pos_lo = P0; tr->pos_hi = P1;
  KMALLOC(ctx, tr->hash, 8 * na, st);
  KMALLOC(ctx, tr->req, 4 * na, st);
  KMALLOC(ctx, tr->prev, 4 * na, st);
  KMALLOC(ctx, tr->delta, 4 * na, st);
  KMALLOC(ctx, tr->depth, 4 * na, st);

  // ---- a2: K1 on the shard (only the shard's token / hash range is uploaded)
  SortedHashes prep;  // K2's sort input, written by K1 in TOKENS mode
  {
    int64_t lo = 0, hi = 0;
    if (r1 > r0 && !d->inputs_on_device) {  // element range covering the shard's requests
      std::vector<int64_t> so(r1 - r0);
      KCUDA(ctx, cudaMemcpyAsync(so.data(), in.src_off.p + r0, 8 * (r1 - r0), cudaMemcpyDeviceToHost, st));
      std::vector<uint64_t> nb(r1 - r0);
      KCUDA(ctx, cudaMemcpyAsync(nb.data(), in.nblk.p + r0, 8 * (r1 - r0), cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      lo = INT64_MAX;
      for (int64_t i = 0; i < r1 - r0; i++) {
        if (nb[i] == 0) continue;
        const int64_t e = so[i] + (int64_t)nb[i] * (d->mode == KARETO_TOKENS ? 16 : 1);
        lo = so[i] < lo ? so[i] : lo;
        hi = e > hi ? e : hi;
      }
      if (lo == INT64_MAX) lo = hi = 0;
    }
    DBuf<uint32_t> h_tok;
    DBuf<uint64_t> h_bh;
    const uint32_t *tok_base;
    const uint64_t *bh_base;
    KTRY(upload_payload(ctx, d, lo, hi, h_tok, h_bh, &tok_base, &bh_base));
    KTRY(chain_hash(ctx, d, tr, in, tok_base, bh_base, d->inputs_on_device ? in.total : hi, r0, r1, tr->hash,
                    tr->req, &prep));
  }

  // ---- a3: in-shard links, then the owner exchange for the shard's first / last accesses
  DBuf<uint32_t> prev_loc;
  DBuf<uint8_t> tmp;
  KTRY(prev_loc.alloc(ctx, na));
  SortedHashes sh;
  DBuf<XRec> rec;
  uint32_t n_rec = 0;
  std::vector<uint64_t> send_cnt(W, 0);
  if (n > 0) KTRY(link_prev(ctx, tr->hash, n, prev_loc.p, &sh, &prep));
  {
    Pass ps(ctx, "F4_records", 1, 3);
    DBuf<uint8_t> fl;
    DBuf<uint32_t> cnt, off;
    KTRY(fl.alloc(ctx, na));
    KTRY(cnt.alloc(ctx, na + 1)); KTRY(off.alloc(ctx, na + 1));
    KCUDA(ctx, cudaMemsetAsync(cnt.p, 0, 4 * (na + 1), st));
    if (n > 0) k_rec_flags<<<grid_for(n, 256, 8 * sms), 256, 0, st>>>(sh.qf.p, sh.nx.p, n, fl.p, cnt.p);
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceScan::ExclusiveSum(t, b, cnt.p, off.p, (int64_t)(n + 1), st);
    }));
    KCUDA(ctx, cudaMemcpyAsync(&n_rec, off.p + n, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    KTRY(rec.alloc(ctx, n_rec > 0 ? n_rec : 1));
    std::vector<uint32_t> ob(W + 1, 0);
    if (n > 0) {
      k_rec_emit<<<grid_for(n, 256, 8 * sms), 256, 0, st>>>(sh.key.p, sh.val.p, n, fl.p, off.p, tr->req, tr->s,
                                                            tr->hash, P0, me, rec.p);
      DBuf<uint32_t> dob;
      KTRY(dob.alloc(ctx, W + 1));
      k_owner_bounds<<<1, 256, 0, st>>>(rec.p, n_rec, W, dob.p);
      KCUDA(ctx, cudaMemcpyAsync(ob.data(), dob.p, 4 * (W + 1), cudaMemcpyDeviceToHost, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
    }
    for (int o = 0; o < W; o++) send_cnt[o] = ob[o + 1] - ob[o];
  }
  sh.key.release();
  sh.val.release();
  sh.qf.release();
  sh.nx.release();
  // record counts: cnt_all[src * W + dst]
  std::vector<uint64_t> cnt_all((size_t)W * W);
  KTRY(coll_allgather_host(ctx, send_cnt.data(), cnt_all.data(), 8 * W));
  std::vector<uint64_t> recv_cnt(W);
  for (int r = 0; r < W; r++) recv_cnt[r] = cnt_all[(size_t)r * W + me];
  const std::vector<size_t> soff = offsets_of(send_cnt, sizeof(XRec)), roff = offsets_of(recv_cnt, sizeof(XRec));
  const uint64_t n_in = roff[W] / sizeof(XRec);
  // every rank checks every rank's incoming count (all know cnt_all), so all fail together and
  // none leaves a peer waiting in the all-to-all below
  for (int d = 0; d < W; d++) {
    uint64_t in_d = 0;
    for (int r = 0; r < W; r++) in_d += cnt_all[(size_t)r * W + d];
    if (in_d >= (uint64_t)kNone) return fail(ctx, KARETO_E_OVERFLOW, "too many exchange records (rank %d)", d);
  }
  DBuf<XRec> inrec;
  KTRY(inrec.alloc(ctx, n_in > 0 ? n_in : 1));
  {
    Pass ps(ctx, "F4_exchange", 0, 1);
    KTRY(coll_alltoallv(ctx, rec.p, soff, inrec.p, roff));
  }

  // ---- owner: answer each Q with the previous shard's P, each P with the next shard
  // [0] chain violations, [1] reuse intervals >= 2^32-1 ms, [2] internal inconsistencies; all
  // ranks learn them from one allreduce and fail together (no rank may leave a collective early)
  DBuf<unsigned long long> flags;
  KTRY(flags.alloc(ctx, 3)); KTRY(flags.zero());
  DBuf<uint32_t> reply;
  KTRY(reply.alloc(ctx, n_in > 0 ? n_in : 1));
  if (n_in > 0) {
    Pass ps(ctx, "F4_owner", 1, 3);
    std::vector<uint64_t> co(W + 1, 0);
    for (int r = 0; r < W; r++) co[r + 1] = co[r] + recv_cnt[r];
    DBuf<uint64_t> dco;
    KTRY(dco.alloc(ctx, W + 1));
    KCUDA(ctx, cudaMemcpyAsync(dco.p, co.data(), 8 * (W + 1), cudaMemcpyHostToDevice, st));
    // keys owned by this rank: {key : owner_of(key) = me} = [ceil(me 2^32 / W), ceil((me+1) 2^32 / W))
    const uint64_t klo = (((uint64_t)me << 32) + W - 1) / W, khi = (((uint64_t)(me + 1) << 32) + W - 1) / W;
    // buckets of 2^shift consecutive keys, ~256-512 records each
    uint32_t Bt = 1;
    while (Bt < (1u << 22) && (uint64_t)Bt * 512 < n_in) Bt <<= 1;
    int shift = 0;
    while (shift < 32 && ((khi - klo + (1ull << shift) - 1) >> shift) > Bt) shift++;
    const uint32_t B = (uint32_t)((khi - klo + (1ull << shift) - 1) >> shift);
    const unsigned g = B < (uint32_t)(64 * sms) ? B : (unsigned)(64 * sms);
    DBuf<uint32_t> bnd;
    KTRY(bnd.alloc(ctx, (size_t)W * (B + 1)));
    k_bucket_bounds_empty<<<grid_for(B + 1, 256, 4 * sms), 256, 0, st>>>(dco.p, W, B, bnd.p);
    k_bucket_bounds<<<grid_for(n_in, 256, 8 * sms), 256, 0, st>>>(inrec.p, dco.p, W, (uint32_t)klo, shift, B,
                                                                   (uint32_t)n_in, bnd.p);
    k_owner<<<g, OWN_THREADS, 0, st>>>(inrec.p, bnd.p, W, B, reply.p, flags.p);
  }
  inrec.release();
  // answers back to the record senders (same segment sizes, reversed)
  DBuf<uint32_t> ans;
  KTRY(ans.alloc(ctx, n_rec > 0 ? n_rec : 1));
  {
    Pass ps(ctx, "F4_exchange", 0, 1);
    KTRY(coll_alltoallv(ctx, reply.p, offsets_of(recv_cnt, 4), ans.p, offsets_of(send_cnt, 4)));
  }
  reply.release();

  // ---- global prev; boundary LRU sets: this shard's contribution to every later rank as a
  // bitmap over its positions, exchanged, OR-assembled into B_k over [0, P0)
  const uint64_t nw = ((uint64_t)P0 + 31) / 32, nwa = nw > 0 ? nw + 1 : 1;
  DBuf<uint32_t> bits, pc, pre, prev_c, first_cnt, reuse_cnt;
  DBuf<uint8_t> run_flag, nxs;
  const int64_t nra = r1 > r0 ? r1 - r0 : 1;
  KTRY(bits.alloc(ctx, nwa)); KTRY(bits.zero()); KTRY(pc.alloc(ctx, nwa)); KTRY(pre.alloc(ctx, nwa));
  KTRY(prev_c.alloc(ctx, na)); KTRY(run_flag.alloc(ctx, na)); KTRY(nxs.alloc(ctx, na)); KTRY(nxs.zero());
  KTRY(first_cnt.alloc(ctx, nra)); KTRY(reuse_cnt.alloc(ctx, nra));
  KTRY(first_cnt.zero()); KTRY(reuse_cnt.zero());
  auto wrange = [&](int j, uint32_t &w0, uint32_t &nwj) {  // word range of shard j's positions
    w0 = sb[j] >> 5;
    nwj = sb[j + 1] > sb[j] ? ((sb[j + 1] + 31) >> 5) - w0 : 0;
  };
  uint32_t mw0, mnw;
  wrange(me, mw0, mnw);
  std::vector<size_t> bso(W + 1, 0), bro(W + 1, 0);
  for (int k = 0; k < W; k++) {
    uint32_t w0, nwj;
    bso[k + 1] = bso[k] + (k > me ? 4 * (size_t)mnw : 0);
    wrange(k, w0, nwj);
    bro[k + 1] = bro[k] + (k < me ? 4 * (size_t)nwj : 0);
  }
  DBuf<uint32_t> bsend, brecv;
  KTRY(bsend.alloc(ctx, bso[W] / 4 + 1)); KTRY(brecv.alloc(ctx, bro[W] / 4 + 1));
  {
    Pass ps(ctx, "F4_boundary_sets", 1, 3);
    if (n > 0) k_prev_global<<<grid_for(n, 256, 8 * sms), 256, 0, st>>>(prev_loc.p, n, P0, tr->prev);
    if (n_rec > 0)
      k_apply_replies<<<grid_for(n_rec, 256, 8 * sms), 256, 0, st>>>(rec.p, ans.p, n_rec, P0, tr->prev, nxs.p);
    if (me + 1 < W && mnw > 0)  // rank k's segment starts at bso[k] = (k - me - 1) * 4 * mnw
      k_bset_words<<<grid_for(32ll * mnw, 256, 8 * sms), 256, 0, st>>>(nxs.p, P0, P1, mw0, mnw, me, W, bsend.p);
  }
  {
    Pass ps(ctx, "F4_exchange", 0, 1);
    KTRY(coll_alltoallv(ctx, bsend.p, bso, brecv.p, bro));
  }
  bsend.release();
  uint32_t Bsize = 0;
  {
    Pass ps(ctx, "F4_boundary", 1, 3);
    for (int j = 0; j < me; j++) {
      uint32_t w0, nwj;
      wrange(j, w0, nwj);
      if (nwj) k_or_words<<<grid_for(nwj, 256, 8 * sms), 256, 0, st>>>(brecv.p + bro[j] / 4, w0, nwj, (uint32_t)nwa,
                                                                         bits.p);
    }
    k_popc<<<grid_for(nwa, 256, 8 * sms), 256, 0, st>>>(bits.p, nwa, pc.p);
    KTRY(cub_run(ctx, tmp, [&](void *t, size_t &b) {
      return cub::DeviceScan::ExclusiveSum(t, b, pc.p, pre.p, (int64_t)nwa, st);
    }));
    uint32_t last[2] = {0, 0};
    KCUDA(ctx, cudaMemcpyAsync(&last[0], pre.p + nwa - 1, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaMemcpyAsync(&last[1], pc.p + nwa - 1, 4, cudaMemcpyDeviceToHost, st));
    KCUDA(ctx, cudaStreamSynchronize(st));
    Bsize = last[0] + last[1];
    if ((uint64_t)Bsize + n >= (1ull << 31)) {
      const unsigned long long one = 1;
      KCUDA(ctx, cudaMemcpyAsync(flags.p + 2, &one, 8, cudaMemcpyHostToDevice, st));
      KCUDA(ctx, cudaStreamSynchronize(st));
      Bsize = 0;
    }
    if (n > 0)
      k_access_info_shard<<<grid_for(n, 256, 8 * sms), 256, 0, st>>>(
          n, P0, (uint32_t)r0, tr->prev, tr->req, tr->s, R, tr->arr, tr->hash, bits.p, pre.p, Bsize, tr->delta,
          prev_c.p, first_cnt.p, reuse_cnt.p, run_flag.p, flags.p);
  }
  rec.release(); ans.release(); brecv.release(); nxs.release(); bits.release(); pc.release(); pre.release();
  prev_loc.release();

  // ---- groups, group tables, U, flags (one allreduce)
  const int K = tr->K, G = K + 1;
  {
    Pass ps(ctx, "F4_groups", 0, 0);  // own launches counted inside
    KTRY(shard_groups(ctx, tr, reuse_cnt.p));
  }
  DBuf<unsigned long long> tab;
  KTRY(tab.alloc(ctx, 2 * G + 3)); KTRY(tab.zero());
  if (r1 > r0) {
    k_group_tables<<<grid_for(r1 - r0, 256, 4 * sms), 256, 16 * G, st>>>(r1 - r0, (uint32_t)r0, tr->grp, first_cnt.p,
                                                                        reuse_cnt.p, tab.p, G);
    ctx->own_launches++;
  }
  KCUDA(ctx, cudaMemcpyAsync(tab.p + 2 * G, flags.p, 24, cudaMemcpyDeviceToDevice, st));
  KTRY(coll_allreduce_u64(ctx, tab.p, 2 * G + 3));
  std::vector<unsigned long long> h(2 * G + 3);
  KCUDA(ctx, cudaMemcpyAsync(h.data(), tab.p, 8 * (2 * G + 3), cudaMemcpyDeviceToHost, st));
  KCUDA(ctx, cudaStreamSynchronize(st));
  tr->U_g.resize(G);
  tr->reuse_g.resize(G);
  int64_t U = 0;
  for (int g = 0; g < G; g++) {
    tr->U_g[g] = (int64_t)h[2 * g];
    tr->reuse_g[g] = (int64_t)h[2 * g + 1];
    U += tr->U_g[g];
  }
  tr->U = U;
  if (h[2 * G]) return fail(ctx, KARETO_E_CHAIN, "block hashes are not chain-consistent (R7)");
  if (h[2 * G + 1]) return fail(ctx, KARETO_E_OVERFLOW, "a reuse interval >= 2^32-1 ms");
  if (h[2 * G + 2]) return fail(ctx, KARETO_E_OVERFLOW, "time shards: boundary LRU set inconsistent or >= 2^31 positions");

  // ---- a4: K3 on the shard prefixed by its boundary LRU stack
  KTRY(stack_depth(ctx, n, (uint64_t)Bsize + n, prev_c.p, tr->req, (uint32_t)r0, tr->s + r0, P0, Bsize, run_flag.p,
                   tr->depth, &tr->n_runs));
  KTRY(sync(ctx, "load_trace_sharded"));
  guard.keep = true;
  *out = tr;
  return KARETO_OK;
}

}  // namespace kareto

extern "C" kareto_status kareto_load_trace_sharded(kareto_ctx *ctx, const kareto_trace_desc *desc,
                                                   kareto_trace **out) {
  if (!ctx || !desc || !out) return KARETO_E_INVALID;
  *out = nullptr;
  ctx->err.clear();
  cudaSetDevice(ctx->device);
  kareto_status s = kareto::load_sharded(ctx, desc, out);
  if (s != KARETO_OK) {
    cudaStreamSynchronize(ctx->stream);
    (void)cudaGetLastError();
  }
  return s;
}

extern "C" kareto_status kareto_trace_shard(const kareto_trace *tr, int64_t *req_lo, int64_t *req_hi, int64_t *pos_lo,
                                            int64_t *pos_hi) {
  if (!tr) return KARETO_E_INVALID;
  if (req_lo) *req_lo = tr->req_lo;
  if (req_hi) *req_hi = tr->req_hi;
  if (pos_lo) *pos_lo = tr->pos_lo;
  if (pos_hi) *pos_hi = tr->pos_hi;
  return KARETO_OK;
}

extern "C" kareto_status kareto_time_slices(const uint32_t *s, int64_t R, int32_t world, int64_t *req_bounds) {
  if (!s || R < 1 || world < 1 || world > kareto::kMaxShardWorld || !req_bounds) return KARETO_E_INVALID;
  for (int k = 0; k <= world; k++) req_bounds[k] = kareto::slice_bound(s, R, (uint64_t)s[R], world, k);
  return KARETO_OK;
}

extern "C" int32_t kareto_hash_owner(uint64_t block_hash, int32_t world) {
  if (world < 1) return -1;
  return (int32_t)kareto::owner_of((uint32_t)(kareto::fmix64(block_hash ^ kareto::kSortMixC) >> 32), world);
}

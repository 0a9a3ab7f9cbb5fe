// bucket_link.cuh -- row a3 (K2): the whole-trace previous-access link over 16-bit buckets.
//
// prev[j] = the largest j' < j touching the same block (the reuse interval
// Delta of P:748-756 and every later step read it).  kareto_load_trace sorts K2's
// (fingerprint, identity | position) pairs by the top BL_BITS fingerprint bits only (two stable
// CUB onesweep passes instead of the four a full 32-bit sort needs): a "bucket" then holds every
// access of the ~U/2^16 blocks whose mixed hash shares those bits, in position order (K1 writes
// the pairs in position order and LSD radix passes are stable).  A bucket is cut into chunks of
// at most BL_CHUNK accesses, and one warp links a chunk in position order, 32 accesses per step:
//   * __match_any_sync on the 64-bit identity m = (key << 32 | value >> 32) (a bijection of the
//     hash) groups the step's equal blocks; a lane's previous access is the next-lower lane of
//     its group, and the group's first lane looks the block up in a warp-private shared-memory
//     open-addressing table (identity -> last position), filled in step order;
//   * the group's last lane then records its position (new identities claim a slot with an
//     atomicCAS, so two new blocks of one step never share a slot);
//   * (position, prev) pairs go to the 2^15-position bucket of the position (one global atomic
//     per pair, issued BL_BATCH steps at a time so their latencies overlap), which
//     k_bucket_assemble turns into prev[] with one coalesced write per 2^15 positions.
// Chunks are independent, so a hot block (10^5 accesses in one bucket) does not serialise one
// warp: in chunk c > 0 the first access of a block has its previous access (if any) in an
// earlier chunk, so it is parked as a pending record instead of a pair, and every chunk of a
// multi-chunk bucket leaves one (identity, last position) record per block.  k_bucket_fixup then
// walks each multi-chunk bucket's chunks in order with one table, answering chunk c's pending
// records from the last positions of chunks < c (a few dozen records per chunk).
// More than `limit` distinct blocks in a chunk (or in a multi-chunk bucket) raises `overflow` and
// finishes that chunk with prev = none (prev stays a valid array); kareto_load_trace reads the flag
// at its next host synchronisation and re-runs the load with the full 32-bit sort + k_link_tile
// (exact either way), so the bucket path needs no host round trip of its own.
#pragma once
#include "internal.cuh"

namespace kareto {

constexpr int BL_BITS = 16, BL_NB = 1 << BL_BITS;
constexpr int BL_WARPS = 16, BL_SLOTS = 1024, BL_LIMIT = BL_SLOTS * 3 / 4, BL_BATCH = 8;
constexpr uint32_t BL_CHUNK = 4096;
// Pair slots: a 2^15-position bucket is split into 2^sl sub-regions by position mod 2^sl, each
// exactly 2^(15-sl) pairs long (one pair per position) with its own append cursor, so the 10^8
// cursor atomics spread over 2^sl times more addresses (fewer same-address collisions at the L2);
// cursors are spaced cstride words apart.  KARETO_BL_SUB / KARETO_BL_CSTRIDE override (measurements).
constexpr uint32_t BL_SUB_LOG2 = 2, BL_CSTRIDE = 1;
// raw cursor atomic of position p (the in-bucket slot is bl_off(p) + this value; the add is kept
// apart so that the atomic's latency overlaps the next batch instead of stalling the issuing one)
__device__ __forceinline__ uint32_t bl_slot(unsigned *cursor, uint32_t p, uint32_t sl, uint32_t cstride) {
  const uint32_t ci = ((p >> 15) << sl) | (p & ((1u << sl) - 1u));
  return atomicAdd(&cursor[(size_t)ci * cstride], 1u);
}
__device__ __forceinline__ uint64_t bl_pair_at(uint32_t p, uint32_t sl, uint32_t slot) {
  return ((uint64_t)(p >> 15) << 15) + ((p & ((1u << sl) - 1u)) << (15 - sl)) + slot;
}
constexpr uint32_t BL_EMPTY = 0xFFFFFFFFu, BL_CLAIM = 0xFFFFFFFEu;
struct BLTable {
  uint64_t key[BL_SLOTS];
  uint32_t pos[BL_SLOTS];
  uint16_t used[BL_SLOTS];
  uint32_t nused, pad;
};

// chunk -> bucket table (one thread per bucket writes its chunks)
__global__ void k_chunk_bucket(const uint32_t *__restrict__ cstart, uint16_t *__restrict__ cbucket) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < BL_NB)
    for (uint32_t w = cstart[b]; w < cstart[b + 1]; w++) cbucket[w] = (uint16_t)b;
}

// bstart[b] = first sorted index with bucket >= b (b <= 2^16), by binary search: 65,537 short
// searches instead of a pass over all N keys
__global__ void k_bucket_bounds_bs(const uint32_t *__restrict__ ks, uint64_t N, uint32_t *__restrict__ bstart) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > BL_NB) return;
  uint64_t lo = 0, hi = N;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((int)(__ldg(&ks[mid]) >> (32 - BL_BITS)) < b) lo = mid + 1; else hi = mid;
  }
  bstart[b] = (uint32_t)lo;
}

// chunks per bucket (>= 1), for the chunk prefix cstart
__global__ void k_bucket_chunks(const uint32_t *__restrict__ bstart, uint32_t *__restrict__ nch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < BL_NB) {
    const uint32_t sz = bstart[b + 1] - bstart[b];
    nch[b] = sz <= BL_CHUNK ? 1u : (sz + BL_CHUNK - 1) / BL_CHUNK;
  }
}

__device__ __forceinline__ void bl_reset(BLTable &T, int lane) {
  const uint32_t nu = T.nused < (uint32_t)BL_SLOTS ? T.nused : (uint32_t)BL_SLOTS;
  if (T.nused >= (uint32_t)BL_SLOTS) {
    for (int q = lane; q < BL_SLOTS; q += 32) T.pos[q] = BL_EMPTY;
  } else {
    for (uint32_t q = lane; q < nu; q += 32) T.pos[T.used[q]] = BL_EMPTY;
  }
  __syncwarp();
  if (lane == 0) T.nused = 0;
  __syncwarp();
}

// lookup of identity m: found position or kNone; slot = its slot or the insertion point
__device__ __forceinline__ uint32_t bl_find(const BLTable &T, uint64_t m, uint32_t &slot, bool &isnew) {
  uint32_t q = (uint32_t)m & (BL_SLOTS - 1);
  for (;;) {
    const uint32_t p = T.pos[q];
    if (p == BL_EMPTY) { isnew = true; slot = q; return kNone; }
    if (p != BL_CLAIM && T.key[q] == m) { isnew = false; slot = q; return p; }
    q = (q + 1) & (BL_SLOTS - 1);
  }
}

// claim a free slot for a new identity m from `slot` on (another new identity of the same step
// may have taken it)
__device__ __forceinline__ uint32_t bl_claim(BLTable &T, uint64_t m, uint32_t slot) {
  uint32_t q = slot;
  while (atomicCAS(&T.pos[q], BL_EMPTY, BL_CLAIM) != BL_EMPTY) q = (q + 1) & (BL_SLOTS - 1);
  T.key[q] = m;
  const uint32_t u = atomicAdd(&T.nused, 1u);
  if (u < BL_SLOTS) T.used[u] = (uint16_t)q;
  return q;
}

// Chunk records (multi-chunk buckets only), both indexed by the chunk's sorted range [s0, s1):
// pending = first accesses of blocks in chunk c > 0 (rec_*), last = one per block of the chunk
// (lst_*); counts rec_n[2w] / rec_n[2w + 1] for chunk w.
__global__ void __launch_bounds__(BL_WARPS * 32) k_bucket_link(
    const uint32_t *__restrict__ ks, const uint64_t *__restrict__ vs, const uint32_t *__restrict__ bstart,
    const uint32_t *__restrict__ cstart, const uint16_t *__restrict__ cbucket, unsigned *__restrict__ next, unsigned *__restrict__ cursor,
    uint2 *__restrict__ pairs, uint64_t *__restrict__ rec_m, uint32_t *__restrict__ rec_p, uint64_t *__restrict__ lst_m,
    uint32_t *__restrict__ lst_p, uint32_t *__restrict__ rec_n, unsigned *__restrict__ overflow, uint32_t limit,
    uint32_t sl, uint32_t cstride) {
  extern __shared__ __align__(16) uint8_t bl_raw[];
  BLTable &T = reinterpret_cast<BLTable *>(bl_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  const uint32_t n_chunks = cstart[BL_NB];
  for (int q = lane; q < BL_SLOTS; q += 32) T.pos[q] = BL_EMPTY;
  if (lane == 0) T.nused = 0;
  __syncwarp();
  for (;;) {
    unsigned w = 0;
    if (lane == 0) w = atomicAdd(next, 1u);
    w = __shfl_sync(0xFFFFFFFFu, w, 0);
    if (w >= n_chunks) break;
    const int b = (int)cbucket[w];  // bucket of chunk w (the last b with cstart[b] <= w)
    const uint32_t c = w - cstart[b], nc = cstart[b + 1] - cstart[b];
    const uint32_t s0 = bstart[b] + c * BL_CHUNK;
    const uint32_t s1 = min(bstart[b + 1], s0 + BL_CHUNK);
    const bool multi = nc > 1;
    uint32_t npend = 0;
    // degraded: the chunk holds more than `limit` distinct blocks -- the overflow flag is raised
    // (the caller re-runs the load with the full sort) and the rest of the chunk is emitted with
    // prev = none, so every position still gets exactly one pair and prev stays a valid array
    bool degraded = false;
    // software pipeline: the next batch's loads are in flight while the current batch is linked,
    // and a batch's pairs are stored after the next batch's steps, so the slot atomics' latency
    // hides behind them
    uint64_t m[BL_BATCH];
    uint32_t pos[BL_BATCH];
    auto load_batch = [&](uint32_t base, uint64_t *mm, uint32_t *pp) {
#pragma unroll
      for (int k = 0; k < BL_BATCH; k++) {
        const uint32_t i = base + 32 * k + lane;
        if (i < s1) {
          const uint64_t v = vs[i];
          mm[k] = ((uint64_t)ks[i] << 32) | (v >> 32);
          pp[k] = (uint32_t)v;
        } else {
          mm[k] = 0;
          pp[k] = BL_EMPTY;
        }
      }
    };
    load_batch(s0, m, pos);
    uint32_t spos[BL_BATCH], sprv[BL_BATCH], sat[BL_BATCH];
#pragma unroll
    for (int k = 0; k < BL_BATCH; k++) spos[k] = BL_EMPTY;
    for (uint32_t base = s0; base < s1; base += 32 * BL_BATCH) {
      uint64_t mn[BL_BATCH];
      uint32_t pn[BL_BATCH], prv[BL_BATCH];
      load_batch(base + 32 * BL_BATCH, mn, pn);
#pragma unroll
      for (int k = 0; k < BL_BATCH; k++) prv[k] = kNone;
      if (!degraded) {
#pragma unroll
        for (int k = 0; k < BL_BATCH; k++) {
          if (base + 32 * k >= s1) break;  // warp-uniform
          const bool in = pos[k] != BL_EMPTY;
          const unsigned act = __ballot_sync(0xFFFFFFFFu, in);
          unsigned peers = 0;
          if (in) peers = __match_any_sync(act, m[k]);
          const unsigned lower = peers & below;
          const bool first = in && lower == 0;
          const bool last = in && (peers >> lane) == 1u;
          uint32_t slot = 0, found = kNone;
          bool isnew = false;
          if (first) found = bl_find(T, m[k], slot, isnew);  // on the state before this step
          __syncwarp();
          if (isnew) slot = bl_claim(T, m[k], slot);
          const int src_first = in ? __ffs(peers) - 1 : lane;
          const int src_prev = lower ? 31 - __clz(lower) : lane;
          const uint32_t gslot = __shfl_sync(0xFFFFFFFFu, slot, src_first);
          const uint32_t ppos = __shfl_sync(0xFFFFFFFFu, pos[k], src_prev);
          __syncwarp();
          if (last) T.pos[gslot] = pos[k];
          if (in) prv[k] = lower ? ppos : found;
          // first access of a block in chunk c > 0: its previous access (if any) is in an
          // earlier chunk -- park it for k_bucket_fixup instead of emitting a pair now
          const bool pend = multi && c > 0 && first && isnew;
          const unsigned pb = __ballot_sync(0xFFFFFFFFu, pend);
          if (pend) {
            const uint32_t at = s0 + npend + __popc(pb & below);
            rec_m[at] = m[k];
            rec_p[at] = pos[k];
            pos[k] = BL_EMPTY;  // no pair from this kernel
          }
          npend += __popc(pb);
          __syncwarp();
        }
        if (T.nused > limit) {  // warp-uniform read after the syncs
          if (lane == 0) atomicOr(overflow, 1u);
          degraded = true;
        }
      }
#pragma unroll
      for (int k = 0; k < BL_BATCH; k++)  // the previous batch's pairs (its atomics have returned)
        if (spos[k] != BL_EMPTY) pairs[bl_pair_at(spos[k], sl, sat[k])] = make_uint2(spos[k], sprv[k]);
#pragma unroll
      for (int k = 0; k < BL_BATCH; k++) {
        sat[k] = pos[k] != BL_EMPTY ? bl_slot(cursor, pos[k], sl, cstride) : 0u;
        spos[k] = pos[k];
        sprv[k] = prv[k];
        m[k] = mn[k];
        pos[k] = pn[k];
      }
    }
#pragma unroll
    for (int k = 0; k < BL_BATCH; k++)
      if (spos[k] != BL_EMPTY) pairs[bl_pair_at(spos[k], sl, sat[k])] = make_uint2(spos[k], sprv[k]);
    if (multi) {
      const uint32_t nu = degraded ? 0u : T.nused;  // a degraded chunk leaves no last positions
      for (uint32_t q = lane; q < nu; q += 32) {
        const uint32_t sl = T.used[q];
        lst_m[s0 + q] = T.key[sl];
        lst_p[s0 + q] = T.pos[sl];
      }
      if (lane == 0) {
        rec_n[2 * (size_t)w] = npend;
        rec_n[2 * (size_t)w + 1] = nu;
      }
    }
    bl_reset(T, lane);
  }
}

// Multi-chunk buckets: one warp walks a bucket's chunks in order with one table (identity -> last
// position in chunks < c), answering chunk c's pending records, then recording its blocks' last
// positions.
__global__ void __launch_bounds__(BL_WARPS * 32) k_bucket_fixup(
    const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ cstart, unsigned *__restrict__ next,
    unsigned *__restrict__ cursor, uint2 *__restrict__ pairs, const uint64_t *__restrict__ rec_m,
    const uint32_t *__restrict__ rec_p, const uint64_t *__restrict__ lst_m, const uint32_t *__restrict__ lst_p,
    const uint32_t *__restrict__ rec_n, unsigned *__restrict__ overflow, uint32_t limit, uint32_t sl,
    uint32_t cstride) {
  extern __shared__ __align__(16) uint8_t bl_raw[];
  BLTable &T = reinterpret_cast<BLTable *>(bl_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < BL_SLOTS; q += 32) T.pos[q] = BL_EMPTY;
  if (lane == 0) T.nused = 0;
  __syncwarp();
  for (;;) {
    unsigned b = 0;
    if (lane == 0) b = atomicAdd(next, 1u);
    b = __shfl_sync(0xFFFFFFFFu, b, 0);
    if (b >= (unsigned)BL_NB) break;
    const uint32_t c0 = cstart[b], nc = cstart[b + 1] - c0;
    if (nc <= 1) continue;
    bool degraded = false;  // table over `limit`: flag raised, remaining pending get prev = none
    for (uint32_t c = 0; c < nc; c++) {
      const uint32_t s0 = bstart[b] + c * BL_CHUNK;
      const uint32_t np = rec_n[2 * (size_t)(c0 + c)], nl = rec_n[2 * (size_t)(c0 + c) + 1];
      for (uint32_t q0 = 0; q0 < np; q0 += 32) {  // pending: lookups only (distinct identities)
        const uint32_t q = q0 + lane;
        if (q < np) {
          const uint64_t m = rec_m[s0 + q];
          const uint32_t p = rec_p[s0 + q];
          uint32_t slot;
          bool isnew;
          const uint32_t prv = degraded ? kNone : bl_find(T, m, slot, isnew);
          const uint32_t at = bl_slot(cursor, p, sl, cstride);
          pairs[bl_pair_at(p, sl, at)] = make_uint2(p, prv);
        }
      }
      __syncwarp();
      for (uint32_t q0 = 0; q0 < (degraded ? 0u : nl); q0 += 32) {  // last positions: insert or overwrite
        const uint32_t q = q0 + lane;
        const bool in = q < nl;
        uint64_t m = 0;
        uint32_t p = 0, slot = 0;
        bool isnew = false;
        if (in) {
          m = lst_m[s0 + q];
          p = lst_p[s0 + q];
          (void)bl_find(T, m, slot, isnew);
        }
        __syncwarp();
        if (in && isnew) slot = bl_claim(T, m, slot);
        __syncwarp();
        if (in) T.pos[slot] = p;
        __syncwarp();
      }
      if (!degraded && T.nused > limit) {
        if (lane == 0) atomicOr(overflow, 1u);
        degraded = true;
      }
    }
    bl_reset(T, lane);
  }
}

}  // namespace kareto

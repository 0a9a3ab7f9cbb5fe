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
// sectors.  The replay is latency-bound (dependent HBM round trips per access), so the
// design minimises round trips and per-configuration bytes (bytes bound the wave size):
//   * configurations are split into four classes {list, LFU} x {expiry heap or not}, each
//     with its own field set, waves sized to free HBM per class;
//   * LRU / FIFO tiers are doubly-linked lists with both links in one 8-byte word, loaded
//     speculatively with the tier byte, so an HBM hit costs one round trip;
//   * LFU tiers are frequency buckets (one list per frequency, ordered by last access; victim =
//     the oldest block of the lowest non-empty bucket, found through a two-level bitmap), the
//     disk-expiry heap is 4-ary with the key stored inline in the slot;
//   * the lookup pass issues its loads sixteen blocks at a time, and the UPDATE pass loads the
//     next block's state while the current one is processed;
//   * head / tail / sizes / counters live in registers.
// Victim order: list tail (LRU: least recent -- a demoted block's recency exceeds every
// member of the lower tier, so demotion order is recency order; FIFO: entry order), LFU heap
// minimum of (freq, last_seq); both keys are unique, so the result never depends on heap shape.
#include "replay.cuh"

#include <algorithm>
#include <array>
#include <map>
#include <vector>

namespace kareto {

enum : uint8_t { T_NONE = 0, T_HBM = 1, T_DRAM = 2, T_DISK = 3 };
constexpr int LOOK = 16;  // LOOKUP blocks whose loads are issued together

struct RState {
  uint8_t *tier;       // [b*W+c] T_*
  uint32_t *lt;        // expiry classes: [b*W+c] ms of the last access (the disk expiry base)
  uint2 *link;         // list classes: [b*W+c] (prev, next) toward head / tail
  uint32_t *freq;      // LFU: [b*W+c] access count of a resident block
  uint32_t *bh[3];     // LFU: [f*W+c] newest block of frequency bucket f per tier
  uint32_t *bt[3];     // LFU: [f*W+c] oldest block of frequency bucket f per tier
  uint64_t *occ[3];    // LFU: [w*W+c] bucket occupancy bitmap (bit f) per tier
  uint64_t *occ2[3];   // LFU: [w2*W+c] summary: bit w set iff occ word w is non-zero
  uint32_t NW, NSW;    // LFU: bitmap words, summary words
  uint2 *elink;        // expiry: [b*W+c] neighbours in the block's expiry list (LRU: its group's
                       // list, newer / older; FIFO / LFU: its wheel bucket, prev / next, where prev
                       // = kHeadMark | bucket for a bucket's first block, kNone = in no bucket)
  uint32_t *eh, *et;   // LRU expiry lists: [g*W+c] newest / oldest disk block of group g
  uint32_t *ebh;       // FIFO / LFU expiry wheel: [k*W+c] first block of bucket k
  uint32_t NB, BSH, a_last;  // wheel: NB buckets of 2^BSH ms covering expiry times <= a_last
  uint8_t *look;       // optional [N][n]: the HBM / DRAM tier each access found at its lookup (the
                       // TTL-mode collapse below), at [position * n + the configuration's index]
  uint64_t look_stride;  // n
  const uint16_t *gblk;
  uint64_t W;
};

// Per-thread replay of one configuration.  Every tier-indexed member is accessed with a
// compile-time tier (template parameter / unrolled cascade), so the per-tier state stays in
// registers rather than local memory.
struct QueueState {  // row f3: per-configuration FCFS queue (DESIGN R50-R53)
  const kareto_model *m;   // kernel-parameter copy
  double *F;               // [I][W] instance free times
  double *ttft;            // [W][R] per-request TTFT
  double bw;               // disk bandwidth of the configuration's medium
  double total;
  uint64_t real, capd;
};

// EXPM: 0 no expiry; 1 expiry heap keyed lt + tau_g; 2 (LRU) one list per group in lt order --
// LRU demotes in recency order, so a group's disk blocks arrive with non-decreasing lt and the
// group's expired blocks are always at its list's old end.
template <bool LFU, int EXPM, bool Q>
struct Rep {
  static constexpr bool EXP = EXPM != 0;
  const RState &v;
  const uint64_t c;
  uint64_t cap[3];
  uint64_t size[3];
  uint32_t head[3], tail[3], tail2[3];
  uint32_t seq;
  bool ttl_mode, lru;
  const uint32_t *tau;
  uint64_t hit[3], miss, evict[3], disk_writes, hit_pos_sum, bytetime, after_hole;
  // prefetched state of the next block of the UPDATE pass; every write to that block's tier /
  // link / heap slot during the current touch is mirrored here, so the copy stays exact
  uint32_t nx = kNone, nx_freq = 0;
  uint32_t minf[3];  // LFU: lowest non-empty frequency bucket per tier
  uint8_t nx_tier = 0;
  uint2 nx_link = make_uint2(0, 0);

  __device__ Rep(const RState &vv, uint64_t cc) : v(vv), c(cc) {}
  __device__ __forceinline__ uint64_t at(uint32_t b) const { return (uint64_t)b * v.W + c; }

  // ------------------------------------------------------------ lists
  // tail2[t] = prev link of tail[t], kept current so an eviction needs no dependent load
  template <int t>
  __device__ __forceinline__ void l_push_front(uint32_t b) {
    const uint32_t h = head[t];
    v.link[at(b)] = make_uint2(kNone, h);
    if (b == nx) nx_link = make_uint2(kNone, h);
    if (h != kNone) {
      v.link[at(h)].x = b;
      if (h == nx) nx_link.x = b;
      if (h == tail[t]) tail2[t] = b;
    } else {
      tail[t] = b;
      tail2[t] = kNone;
    }
    head[t] = b;
  }
  template <int t>
  __device__ __forceinline__ void l_unlink(uint2 lk) {  // lk = link of the removed block
    if (lk.x != kNone) {
      v.link[at(lk.x)].y = lk.y;
      if (lk.x == nx) nx_link.y = lk.y;
    } else {
      head[t] = lk.y;
    }
    if (lk.y != kNone) {
      v.link[at(lk.y)].x = lk.x;
      if (lk.y == nx) nx_link.x = lk.x;
      if (lk.y == tail[t]) tail2[t] = lk.x;
    } else {
      tail[t] = lk.x;
      tail2[t] = lk.x != kNone ? v.link[at(lk.x)].x : kNone;
    }
  }
  template <int t>
  __device__ __forceinline__ uint32_t l_pop_tail() {
    const uint32_t x = tail[t], p = tail2[t];
    if (p != kNone) {
      v.link[at(p)].y = kNone;
      if (p == nx) nx_link.y = kNone;
      tail2[t] = v.link[at(p)].x;  // consumed at the next eviction from this tier
    } else {
      head[t] = kNone;
      tail2[t] = kNone;
    }
    tail[t] = p;
    return x;
  }

  // ------------------------------------------------------------ LFU frequency buckets
  // Each tier keeps one doubly-linked list per frequency, newest block at the front.  A block
  // enters a bucket with a last_seq larger than every member's (HBM: it was just touched; DRAM /
  // disk: victims of one frequency leave the tier above in increasing last_seq), so every bucket
  // is ordered by last_seq and the policy victim -- the smallest (freq, last_seq) -- is the tail
  // of the lowest non-empty bucket.  O(1) per operation except finding the next non-empty
  // bucket, a two-level bitmap scan.
  template <int t>
  __device__ __forceinline__ void bit_set(uint32_t f) {
    const uint64_t w = f >> 6;
    const uint64_t old = v.occ[t][w * v.W + c];
    if (!old) v.occ2[t][(w >> 6) * v.W + c] |= 1ull << (w & 63);
    v.occ[t][w * v.W + c] = old | (1ull << (f & 63));
  }
  template <int t>
  __device__ __forceinline__ void bit_clear(uint32_t f) {
    const uint64_t w = f >> 6;
    const uint64_t nw = v.occ[t][w * v.W + c] & ~(1ull << (f & 63));
    v.occ[t][w * v.W + c] = nw;
    if (!nw) v.occ2[t][(w >> 6) * v.W + c] &= ~(1ull << (w & 63));
  }
  // smallest non-empty frequency >= from (kNone if none)
  template <int t>
  __device__ uint32_t next_set(uint32_t from) const {
    uint64_t w = from >> 6;
    if (w < v.NW) {
      const uint64_t word = v.occ[t][w * v.W + c] & (~0ull << (from & 63));
      if (word) return (uint32_t)((w << 6) + __ffsll((long long)word) - 1);
    }
    const uint64_t w1 = w + 1;
    for (uint64_t sw = w1 >> 6; sw < v.NSW; sw++) {
      uint64_t sm = v.occ2[t][sw * v.W + c];
      if (sw == (w1 >> 6)) sm &= (w1 & 63) ? (~0ull << (w1 & 63)) : ~0ull;
      if (sm) {
        const uint64_t wn = (sw << 6) + __ffsll((long long)sm) - 1;
        return (uint32_t)((wn << 6) + __ffsll((long long)v.occ[t][wn * v.W + c]) - 1);
      }
    }
    return kNone;
  }
  template <int t>
  __device__ __forceinline__ void b_push(uint32_t b, uint32_t f) {
    uint32_t *bh = v.bh[t], *bt = v.bt[t];
    const uint32_t h = bh[(uint64_t)f * v.W + c];
    v.link[at(b)] = make_uint2(kNone, h);
    if (b == nx) nx_link = make_uint2(kNone, h);
    if (h != kNone) {
      v.link[at(h)].x = b;
      if (h == nx) nx_link.x = b;
    } else {
      bt[(uint64_t)f * v.W + c] = b;
      bit_set<t>(f);
    }
    bh[(uint64_t)f * v.W + c] = b;
    if (size[t] == 0 || f < minf[t]) minf[t] = f;
    size[t]++;
  }
  // unlink b (links lk) from bucket f; returns true when the bucket became empty
  template <int t>
  __device__ __forceinline__ bool b_unlink(uint2 lk, uint32_t f, bool fix_min) {
    uint32_t *bh = v.bh[t], *bt = v.bt[t];
    if (lk.x != kNone) {
      v.link[at(lk.x)].y = lk.y;
      if (lk.x == nx) nx_link.y = lk.y;
    } else {
      bh[(uint64_t)f * v.W + c] = lk.y;
    }
    if (lk.y != kNone) {
      v.link[at(lk.y)].x = lk.x;
      if (lk.y == nx) nx_link.x = lk.x;
    } else {
      bt[(uint64_t)f * v.W + c] = lk.x;
    }
    size[t]--;
    const bool empty = lk.x == kNone && lk.y == kNone;
    if (empty) {
      bit_clear<t>(f);
      if (fix_min && f == minf[t] && size[t] > 0) minf[t] = next_set<t>(f + 1);
    }
    return empty;
  }

  // ------------------------------------------------------------ expiry wheel (FIFO / LFU)
  // A disk block with a finite TTL expires at e = lt + tau_g (ms).  Blocks with e <= a_last sit in
  // bucket e >> BSH of a per-configuration wheel (a doubly-linked list per bucket); later ones
  // never expire within the trace.  PURGE(a) empties every bucket below a >> BSH (all their
  // blocks have e < a) and scans the boundary bucket a >> BSH with exact keys.  Buckets below the
  // current boundary pcur are empty; a block inserted with such an e (it expired before it was
  // demoted) goes into the boundary bucket.  O(1) insert / remove, unlike a heap's log-depth
  // chain of dependent loads.  The order of removals inside one PURGE does not change the state.
  uint32_t pcur = 0;
  uint64_t gmin = ~0ull;  // expiry classes: a lower bound of the earliest disk expiry (PURGE skipped
                          // while gmin >= a: removals only raise the true minimum)
  static constexpr uint32_t kHeadMark = 0x80000000u;
  __device__ __forceinline__ void w_push(uint32_t b, uint32_t k) {
    const uint64_t hi = (uint64_t)k * v.W + c;
    const uint32_t h = v.ebh[hi];
    v.elink[at(b)] = make_uint2(kHeadMark | k, h);
    if (h != kNone) v.elink[at(h)].x = b;
    v.ebh[hi] = b;
  }
  __device__ __forceinline__ void w_unlink(uint32_t b) {
    const uint2 lk = v.elink[at(b)];
    if (lk.x == kNone) return;
    if (lk.x & kHeadMark) v.ebh[(uint64_t)(lk.x & ~kHeadMark) * v.W + c] = lk.y;
    else v.elink[at(lk.x)].y = lk.y;
    if (lk.y != kNone) v.elink[at(lk.y)].x = lk.x;
  }
  __device__ __forceinline__ void w_insert(uint32_t b, uint32_t tg) {
    const uint64_t e = (uint64_t)v.lt[at(b)] + tg;
    if (e > v.a_last) {  // never expires within the trace
      v.elink[at(b)] = make_uint2(kNone, kNone);
      return;
    }
    const uint32_t k = (uint32_t)(e >> v.BSH);
    w_push(b, k < pcur ? pcur : k);
    if (e < gmin) gmin = e;
  }
  // drop disk block x (expired): out of the disk tier (the wheel is handled by the caller)
  __device__ __forceinline__ void w_drop(uint32_t x) {
    if (LFU) {
      b_unlink<2>(v.link[at(x)], v.freq[at(x)], true);
    } else {
      l_unlink<2>(v.link[at(x)]);
      size[2]--;
    }
    v.tier[at(x)] = T_NONE;
  }
  __device__ void w_purge(uint32_t a) {
    const uint32_t ka = a >> v.BSH;  // a <= a_last, so ka < NB
    for (; pcur < ka; pcur++) {       // whole buckets: every e < (pcur + 1) << BSH <= a
      const uint64_t hi = (uint64_t)pcur * v.W + c;
      for (uint32_t x = v.ebh[hi]; x != kNone;) {
        const uint32_t nxt = v.elink[at(x)].y;
        w_drop(x);
        x = nxt;
      }
      v.ebh[hi] = kNone;
    }
    const uint64_t hi = (uint64_t)ka * v.W + c;  // boundary bucket: exact keys
    gmin = (uint64_t)(ka + 1) << v.BSH;           // every later bucket expires at or after this
    for (uint32_t x = v.ebh[hi]; x != kNone;) {
      const uint32_t nxt = v.elink[at(x)].y;
      const uint64_t e = (uint64_t)v.lt[at(x)] + tau[v.gblk[x]];
      if (e < a) {
        w_unlink(x);
        w_drop(x);
      } else if (e < gmin) {
        gmin = e;
      }
      x = nxt;
    }
  }

  // ------------------------------------------------------------ tiers (t = 0, 1, 2)
  // insert b (not resident) into tier t; key = LFU key
  template <int t>
  __device__ __forceinline__ void t_insert(uint32_t b, uint64_t key) {
    v.tier[at(b)] = (uint8_t)(t + 1);
    if (b == nx) nx_tier = (uint8_t)(t + 1);
    if (LFU) {
      const uint32_t f = (uint32_t)(key >> 32);
      v.freq[at(b)] = f;
      if (b == nx) nx_freq = f;
      b_push<t>(b, f);
    } else {
      l_push_front<t>(b);
      size[t]++;
    }
    if (EXP && t == 2) {
      const uint16_t g = v.gblk[b];
      const uint32_t tg = tau[g];
      if (tg != KARETO_TTL_INF) {
        if (EXPM == 1) {
          w_insert(b, tg);
        } else {  // newest end of the group's list
          const uint64_t e = (uint64_t)v.lt[at(b)] + tg;
          if (e < gmin) gmin = e;  // keeps gmin a lower bound of every group's oldest expiry
          const uint64_t gi = (uint64_t)g * v.W + c;
          const uint32_t h = v.eh[gi];
          v.elink[at(b)] = make_uint2(kNone, h);
          if (h != kNone) v.elink[at(h)].x = b; else v.et[gi] = b;
          v.eh[gi] = b;
        }
      }
    }
  }
  // remove disk block b from its group's expiry list (EXPM 2)
  __device__ __forceinline__ void ge_remove(uint32_t b) {
    const uint16_t g = v.gblk[b];
    if (tau[g] == KARETO_TTL_INF) return;
    const uint64_t gi = (uint64_t)g * v.W + c;
    const uint2 lk = v.elink[at(b)];
    if (lk.x != kNone) v.elink[at(lk.x)].y = lk.y; else v.eh[gi] = lk.y;
    if (lk.y != kNone) v.elink[at(lk.y)].x = lk.x; else v.et[gi] = lk.x;
  }
  // remove resident b (link / heap slot already loaded) from tier t
  template <int t>
  __device__ __forceinline__ uint64_t t_remove(uint32_t b, uint2 lk, uint32_t fb) {
    uint64_t key = 0;
    if (LFU) {  // fb = the block's frequency
      b_unlink<t>(lk, fb, true);
      key = (uint64_t)fb << 32;
    } else {
      l_unlink<t>(lk);
      size[t]--;
    }
    if (EXPM == 1 && t == 2 && tau[v.gblk[b]] != KARETO_TTL_INF) w_unlink(b);
    if (EXPM == 2 && t == 2) ge_remove(b);
    return key;
  }
  // one CASCADE level: tier t overflows by at most one block; returns false when done
  template <int t>
  __device__ __forceinline__ bool overflow() {
    const uint64_t capt = (t == 2 && ttl_mode) ? 0 : cap[t];
    if (size[t] <= capt) return false;
    uint32_t x;
    uint64_t key = 0;
    if (LFU) {  // the oldest block of the lowest non-empty bucket
      const uint32_t f = minf[t];
      x = v.bt[t][(uint64_t)f * v.W + c];
      b_unlink<t>(v.link[at(x)], f, true);
      key = (uint64_t)f << 32;
    } else {
      x = l_pop_tail<t>();
      size[t]--;
    }
    if (EXPM == 1 && t == 2 && tau[v.gblk[x]] != KARETO_TTL_INF) w_unlink(x);
    if (EXPM == 2 && t == 2) ge_remove(x);
    evict[t] += 1;
    const bool next = ttl_mode ? (t == 0) : (t < 2);
    if (!next) {
      v.tier[at(x)] = T_NONE;
      if (x == nx) nx_tier = T_NONE;
      return false;
    }
    seq += 1;
    if (t < 2) t_insert<(t < 2 ? t + 1 : 2)>(x, key);  // LFU key (freq, last_seq) carried
    return true;
  }
  __device__ __forceinline__ void cascade() {
    if (overflow<0>() && overflow<1>()) overflow<2>();
  }

  // ------------------------------------------------------------ f3 queue (R50-R52)
  QueueState *qs = nullptr;
  __device__ void q_wait(uint32_t a, int &bi, double &start, double &w, double &x) const {
    const double a_s = (double)a * 1e-3;
    const int I = qs->m->instances;
    double fb = qs->F[c];
    bi = 0;
    for (int i = 1; i < I; i++) {
      const double f = qs->F[(size_t)i * v.W + c];
      if (f < fb) { fb = f; bi = i; }
    }
    start = a_s > fb ? a_s : fb;
    w = start - a_s;
    x = (w * qs->bw) / (double)qs->m->block_bytes;
  }
  __device__ void q_serve(const ReplayTrace &T, uint32_t r, int bi, double start, double w, uint64_t H, uint64_t h2,
                          uint64_t nd) {
    const kareto_model &m = *qs->m;
    const uint64_t L = T.inlen[r];
    const uint64_t P0 = m.alpha_ps * L + m.beta_ps * (L * (L - 1) / 2);
    const uint64_t S = 16 * m.alpha_ps * H + m.beta_ps * (256 * (H * (H - 1) / 2) + 120 * H);
    const double prefill = (double)(P0 - S) * 1e-12;
    const double dram = (double)(h2 * m.block_bytes) / m.bw_dram;
    const double decode = (double)(m.dec_ps * (uint64_t)T.outlen[r]) * 1e-12;
    const double t = (w + prefill) + dram;
    qs->total = qs->total + t;
    qs->ttft[(size_t)c * T.R + r] = t;
    qs->F[(size_t)bi * v.W + c] = ((start + prefill) + dram) + decode;
    qs->capd += nd;
  }
  __device__ void q_step(const ReplayTrace &T, uint32_t r, uint32_t a, uint64_t H, uint64_t h2, uint64_t nd,
                         uint64_t) {
    int bi;
    double start, w, x;
    q_wait(a, bi, start, w, x);
    q_serve(T, r, bi, start, w, H, h2, nd);
  }

  __device__ void run(const ReplayTrace &T, const kareto_config &cf, const uint32_t *rows, int n_tuner, int G,
                      kareto_counts *out, QueueState *qsp = nullptr, uint8_t *look = nullptr, uint32_t lstride = 0) {
    qs = qsp;
    cap[0] = cf.cap[0];
    cap[1] = cf.cap[1];
    cap[2] = cf.cap[2];
    lru = cf.policy == KARETO_LRU;
    ttl_mode = cf.cap[2] == KARETO_INF;
    tau = rows + (size_t)(n_tuner > 0 ? cf.tuner : 0) * G;
    bool any_finite = false;
    for (int g = 0; g < G; g++) any_finite |= tau[g] != KARETO_TTL_INF;
#pragma unroll
    for (int t = 0; t < 3; t++) {
      head[t] = tail[t] = tail2[t] = kNone;
      size[t] = 0;
      minf[t] = kNone;
      hit[t] = evict[t] = 0;
    }
    miss = disk_writes = hit_pos_sum = bytetime = after_hole = 0;
    pcur = 0;
    gmin = ~0ull;
    seq = 0;
    uint32_t s0 = T.s[0];
    for (uint32_t r = 0; r < T.R; r++) {
      const uint32_t s1 = T.s[r + 1];
      const uint32_t nb = s1 - s0;
      const uint32_t a = T.arr[r];
      if (nb == 0) {
        if (Q) q_step(T, r, a, 0, 0, 0, 0);  // a request without full blocks still queues
        continue;
      }
      const uint32_t tg = tau[T.grp[r]];
      // 1 PURGE (CAPACITY mode): disk blocks whose expiry key is below a (a - lt > tau_g)
      if (EXPM == 1 && size[2] > 0 && gmin < a) w_purge(a);
      // each group's expired blocks sit at its list's old end; gmin (a lower bound of the earliest
      // expiry over the groups: removals only raise the true minimum) skips the G list probes
      // while nothing can have expired, and is recomputed exactly after a scan
      if (EXPM == 2 && size[2] > 0 && gmin < a) {
        gmin = ~0ull;
        for (int g = 0; g < G; g++) {
          const uint32_t tgg = tau[g];
          if (tgg == KARETO_TTL_INF) continue;
          const uint64_t gi = (uint64_t)g * v.W + c;
          for (uint32_t x = v.et[gi]; x != kNone; x = v.et[gi]) {
            if ((uint64_t)v.lt[at(x)] + tgg >= a) break;
            const uint32_t nxt = v.elink[at(x)].x;  // next older-to-newer
            v.et[gi] = nxt;
            if (nxt != kNone) v.elink[at(nxt)].y = kNone; else v.eh[gi] = kNone;
            l_unlink<2>(v.link[at(x)]);
            size[2]--;
            v.tier[at(x)] = T_NONE;
          }
          const uint32_t y = v.et[gi];
          if (y != kNone) {
            const uint64_t e = (uint64_t)v.lt[at(y)] + tgg;
            if (e < gmin) gmin = e;
          }
        }
      }
      // f3 queue (R50): wait of this request before its lookup; x = disk blocks loadable (R51)
      int qbi = 0;
      double qstart = 0.0, qw = 0.0, qx = 0.0;
      uint64_t qH = 0, qh2 = 0, qnd = 0;
      bool qopen = true;
      if (Q) q_wait(a, qbi, qstart, qw, qx);
      // 2 LOOKUP on the pre-request state: block k sits at position s0 + nb - 1 - k
      bool in_prefix = true;
      for (uint32_t k0 = 0; k0 < nb; k0 += LOOK) {
        uint32_t bb[LOOK];
        uint8_t tt[LOOK];
        uint32_t dd[LOOK];
        // the lease store's state is the trace's: alive iff seen before and delta <= tau_g (the
        // reuse interval of the access is a - the block's last access)
#pragma unroll
        for (int q = 0; q < LOOK; q++) {
          const bool ok = k0 + q < nb;
          bb[q] = ok ? T.blk[s1 - 1 - (k0 + q)] : 0u;
          dd[q] = (ok && ttl_mode) ? T.delta[s1 - 1 - (k0 + q)] : kNone;
        }
#pragma unroll
        for (int q = 0; q < LOOK; q++) tt[q] = k0 + q < nb ? v.tier[at(bb[q])] : 0;
        if (look) {
#pragma unroll
          for (int q = 0; q < LOOK; q++)
            if (k0 + q < nb) look[(size_t)(s1 - 1 - (k0 + q)) * lstride] = tt[q];
        }
#pragma unroll
        for (int q = 0; q < LOOK; q++) {
          if (k0 + q >= nb) break;
          const uint8_t t = tt[q];
          const bool alive = dd[q] != kNone && dd[q] <= tg;
          const bool present = t != T_NONE || (ttl_mode && alive);
          in_prefix = in_prefix && present;
          if (in_prefix) {
            hit[0] += t == T_HBM;
            hit[1] += t == T_DRAM;
            hit[2] += t == T_DISK || t == T_NONE;
            hit_pos_sum += k0 + q;
            if (Q) {  // R51: disk blocks stream in chain order; the first one not loaded ends the prefix
              const bool disk = t == T_DISK || t == T_NONE;
              if (disk) {
                qnd++;
                if (qopen && (double)qnd > qx) qopen = false;
              }
              if (qopen) {
                qH++;
                qh2 += t == T_DRAM;
                qs->real += disk;
              }
            }
          } else {
            miss += 1;
            after_hole += t != T_NONE;
          }
          disk_writes += ttl_mode && !alive;
        }
      }
      if (Q) q_serve(T, r, qbi, qstart, qw, qH, qh2, qnd);
      // 3 UPDATE leaf -> root = touch positions s0 .. s1-1 in order; the state of block j+1 is
      // loaded while block j is processed (mirrored writes keep it exact)
      uint32_t bn = T.blk[s0];
      uint32_t bnn = s0 + 1 < s1 ? T.blk[s0 + 1] : 0u;
      uint8_t t_n = v.tier[at(bn)];
      uint2 lk_n = v.link[at(bn)];
      uint32_t hp_n = LFU ? v.freq[at(bn)] : 0u;
      for (uint32_t j = s0; j < s1; j++) {
        const uint32_t b = bn;
        const uint8_t t = t_n;
        const uint2 lk = lk_n;
        const uint32_t hp = hp_n;
        seq += 1;
        if (j + 1 < s1) {
          bn = bnn;
          if (j + 2 < s1) bnn = T.blk[j + 2];
          nx = bn;
          nx_tier = v.tier[at(bn)];
          nx_link = v.link[at(bn)];
          if (LFU) nx_freq = v.freq[at(bn)];
        } else {
          nx = kNone;
        }
        if (ttl_mode) {  // lease integral since the previous access
          const uint32_t dt = T.delta[j];
          if (dt != kNone) bytetime += dt < tg ? dt : tg;
        }
        if (EXP) v.lt[at(b)] = a;  // expiry base; before any expiry insertion of b in its own cascade
        if (t == T_HBM) {
          if (LFU) {  // move to the front of bucket f + 1
            const uint32_t f = hp;
            const bool emptied = b_unlink<0>(lk, f, false);
            v.freq[at(b)] = f + 1;
            b_push<0>(b, f + 1);
            if (emptied && minf[0] == f) minf[0] = f + 1;
          } else if (lru && head[0] != b) {
            l_unlink<0>(lk);
            l_push_front<0>(b);
          }
        } else {
          uint64_t freq = 1;
          if (t == T_DRAM) freq = (t_remove<1>(b, lk, hp) >> 32) + 1;  // LFU count carried
          else if (t == T_DISK) freq = (t_remove<2>(b, lk, hp) >> 32) + 1;
          t_insert<0>(b, (freq << 32) | seq);
          cascade();
        }
        t_n = nx_tier;
        lk_n = nx_link;
        hp_n = nx_freq;
      }
      s0 = s1;
    }
    if (ttl_mode) {  // every block's last lease counts a full tau (R21): sum_g U_g tau_g
      for (int g = 0; g < G; g++) bytetime += T.Ug[g] * (uint64_t)tau[g];
      evict[2] = 0;
    } else {
      disk_writes = cap[2] > 0 ? evict[1] : 0;
      if (any_finite) evict[2] = KARETO_NA;
    }
    kareto_counts k;
    for (int t = 0; t < 3; t++) { k.hit[t] = hit[t]; k.evict[t] = evict[t]; }
    k.miss = miss;
    k.disk_writes = disk_writes;
    k.hit_pos_sum = hit_pos_sum;
    k.bytetime_block_ms = bytetime;
    k.resident_after_hole = after_hole;
    *out = k;
  }
};

struct QueueKernelArgs {  // row f3 inside the replay (Q = true)
  kareto_model m;
  double *F;                     // [I][W]
  double *ttft;                  // [W][R]
  kareto_queue_result *out;      // indexed by the caller's configuration id
  uint64_t span_ms, LO;
};

template <bool LFU, int EXPM, bool Q>
__global__ void __launch_bounds__(64) k_replay(ReplayTrace T, const kareto_config *__restrict__ cfg,
                                               const uint32_t *__restrict__ idx, const uint32_t *__restrict__ rows,
                                               int n_tuner, int G, RState v, int64_t n,
                                               kareto_counts *__restrict__ out, QueueKernelArgs qa) {
  const int64_t ci = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ci >= n) return;
  const uint32_t id = idx[ci];
  const kareto_config cf = cfg[id];
  Rep<LFU, EXPM, Q> rp(v, (uint64_t)ci);
  if (!Q) {
    rp.run(T, cf, rows, n_tuner, G, out + id, nullptr, v.look ? v.look + id : nullptr, (uint32_t)v.look_stride);
    return;
  }
  QueueState qs;
  qs.m = &qa.m;
  qs.F = qa.F;
  qs.ttft = qa.ttft;
  const bool ttl = cf.cap[2] == KARETO_INF;
  const kareto_medium md = qa.m.media[cf.medium];
  const double prov_gb = ttl ? qa.m.ttl_prov_gb : (double)(cf.cap[2] * qa.m.block_bytes) / 1e9;
  const double bwv = md.bw_base + md.bw_slope * prov_gb;
  qs.bw = md.bw_max < bwv ? md.bw_max : bwv;
  qs.total = 0.0;
  qs.real = qs.capd = 0;
  for (int i = 0; i < qa.m.instances; i++) qa.F[(size_t)i * v.W + ci] = 0.0;
  rp.run(T, cf, rows, n_tuner, G, out + id, &qs);
  double fmax = qa.F[ci];
  for (int i = 1; i < qa.m.instances; i++) {
    const double f = qa.F[(size_t)i * v.W + ci];
    fmax = fmax > f ? fmax : f;
  }
  const double span_s = (double)qa.span_ms * 1e-3;
  const double M = span_s > fmax ? span_s : fmax;
  kareto_queue_result q;
  q.ttft_mean_ms = 1e3 * (qs.total / (double)T.R);
  q.ttft_p99_ms = 0.0;
  q.makespan_s = M;
  q.tokens_per_s = (double)qa.LO / M;
  q.disk_hits_capacity = qs.capd;
  q.disk_hits_realized = qs.real;
  qa.out[id] = q;
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
  KMALLOC(ctx, tr->blk, 4 * N, st);
  KMALLOC(ctx, tr->gblk, 2 * (size_t)(tr->U > 0 ? tr->U : 1), st);
  KMALLOC(ctx, tr->arr_rel, 4 * (size_t)tr->R, st);
  k_dense_ids<<<grid_for(N, 256, 8 * sms), 256, 0, st>>>(N, f0.p, idf.p, tr->prev, tr->req, tr->grp, tr->blk, tr->gblk);
  k_arr_rel<<<grid_for(tr->R, 256, 4 * sms), 256, 0, st>>>(tr->R, tr->arr, tr->arr_rel);
  return KARETO_OK;
}

__global__ void k_pick_p99_idx(const double *__restrict__ sorted, int64_t R, int64_t n, int64_t k,
                               const uint32_t *__restrict__ idx, kareto_queue_result *__restrict__ out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n) out[idx[c]].ttft_p99_ms = 1e3 * sorted[(size_t)c * R + (k - 1)];
}
__global__ void k_row_offsets(int64_t n, int64_t R, int64_t *__restrict__ off) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c <= n) off[c] = c * R;
}

// TTL-mode collapse (FIFO / LFU): with c3 = infinity the disk is the write-through lease store,
// whose state is the trace's own (alive iff delta <= tau_g), and the HBM / DRAM replay never looks
// at it (DRAM victims are dropped; LFU frequencies restart after a drop whatever the lease).  So
// every TTL-mode configuration of one (policy, c1, c2) sees the same HBM / DRAM tier at every
// lookup; one replay per (policy, c1, c2) records them (look) and each member configuration's
// counts follow from (tier, delta, group) per access, for its own TTL row (R9-R22 as in K6).
__global__ void k_ttl_member_counts(ReplayTrace T, const kareto_config *__restrict__ cfg,
                                    const uint32_t *__restrict__ mrep, const uint32_t *__restrict__ mout, int64_t nm,
                                    const uint8_t *__restrict__ look, uint32_t nrep,
                                    const kareto_counts *__restrict__ rep_counts,
                                    const uint32_t *__restrict__ rows, int n_tuner, int G,
                                    kareto_counts *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nm) return;
  const kareto_config cf = cfg[i];
  const uint32_t *tau = rows + (size_t)(n_tuner > 0 ? cf.tuner : 0) * G;
  const uint8_t *lk = look + mrep[i];  // [position * nrep + representative]
  uint64_t hit[3] = {0, 0, 0}, miss = 0, hps = 0, after = 0, dw = 0, bt = 0;
  uint32_t s0 = T.s[0];
  for (uint32_t r = 0; r < T.R; r++) {
    const uint32_t s1 = T.s[r + 1];
    const uint32_t nb = s1 - s0;
    if (nb == 0) continue;
    const uint32_t tg = tau[T.grp[r]];
    bool in_prefix = true;
    for (uint32_t k = 0; k < nb; k++) {
      const uint32_t pos = s1 - 1 - k;
      const uint8_t t = lk[(size_t)pos * nrep];
      const uint32_t dl = T.delta[pos];
      const bool alive = dl != kNone && dl <= tg;
      in_prefix = in_prefix && (t != T_NONE || alive);
      if (in_prefix) {
        hit[0] += t == T_HBM;
        hit[1] += t == T_DRAM;
        hit[2] += t == T_NONE;
        hps += k;
      } else {
        miss += 1;
        after += t != T_NONE;
      }
      dw += !alive;
      if (dl != kNone) bt += dl < tg ? dl : tg;
    }
    s0 = s1;
  }
  for (int g = 0; g < G; g++) bt += T.Ug[g] * (uint64_t)tau[g];  // every block's last lease (R21)
  const kareto_counts &rc = rep_counts[mrep[i]];
  kareto_counts k;
  for (int t = 0; t < 3; t++) k.hit[t] = hit[t];
  k.miss = miss;
  k.evict[0] = rc.evict[0];
  k.evict[1] = rc.evict[1];
  k.evict[2] = 0;
  k.disk_writes = dw;
  k.hit_pos_sum = hps;
  k.bytetime_block_ms = bt;
  k.resident_after_hole = after;
  out[mout[i]] = k;
}

__global__ void k_scatter_counts(const kareto_counts *__restrict__ in, const uint32_t *__restrict__ to, int64_t n,
                                 kareto_counts *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[to[i]] = in[i];
}

kareto_status replay_eval(kareto_ctx *ctx, kareto_trace *tr, const kareto_config *cfg_host, int64_t n,
                          const uint32_t *rows_host, const uint32_t *rows_dev, int n_tuner,
                          kareto_counts *counts_dev, const QueueArgs &qarg, uint8_t *look_dev) {
  if (n <= 0) return KARETO_OK;
  if (qarg.model == nullptr && look_dev == nullptr && getenv("KARETO_K6_NO_COLLAPSE") == nullptr) {
    // TTL-mode collapse (k_ttl_member_counts): one replay per (policy, c1, c2) group of TTL-mode
    // FIFO / LFU configurations, when that saves at least half of their replays and the lookup
    // record fits in a quarter of the free device memory
    std::map<std::array<uint64_t, 3>, std::vector<int64_t>> grp;
    for (int64_t i = 0; i < n; i++) {
      const kareto_config &c = cfg_host[i];
      if (c.cap[2] == KARETO_INF && (c.policy == KARETO_FIFO || c.policy == KARETO_LFU))
        grp[{(uint64_t)c.policy, c.cap[0], c.cap[1]}].push_back(i);
    }
    int64_t nmem = 0;
    for (auto &kv : grp) nmem += (int64_t)kv.second.size();
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const uint64_t Nn = (uint64_t)tr->N;
    // worth it when the members alone would not fit one wave (a full-size grid: their replays are
    // whole extra passes over the trace); with room to spare (a small trace) they ride along with
    // the other classes' concurrent waves for free and the collapse would add a pass
    const double member_bytes = (double)nmem * (double)(tr->U > 0 ? tr->U : 1) * 13.0;
    const bool force = getenv("KARETO_K6_COLLAPSE") != nullptr;
    if (!grp.empty() && nmem >= 2 * (int64_t)grp.size() && (double)grp.size() * (double)Nn <= 0.25 * (double)fr &&
        (force || member_bytes > 0.8 * (double)fr)) {
      const int64_t nrep = (int64_t)grp.size();
      std::vector<kareto_config> reps, mcfg, rest;
      std::vector<uint32_t> mrep, mout, rout;
      std::vector<char> collapsed((size_t)n, 0);
      for (auto &kv : grp) {
        const uint32_t ri = (uint32_t)reps.size();
        reps.push_back(cfg_host[kv.second[0]]);
        for (int64_t i : kv.second) {
          collapsed[(size_t)i] = 1;
          mcfg.push_back(cfg_host[i]);
          mrep.push_back(ri);
          mout.push_back((uint32_t)i);
        }
      }
      for (int64_t i = 0; i < n; i++)
        if (!collapsed[(size_t)i]) { rest.push_back(cfg_host[i]); rout.push_back((uint32_t)i); }
      DBuf<uint8_t> look;
      DBuf<kareto_counts> rcnt;
      KTRY(look.alloc(ctx, (size_t)nrep * (Nn > 0 ? Nn : 1)));
      KTRY(rcnt.alloc(ctx, nrep));
      KTRY(replay_eval(ctx, tr, reps.data(), nrep, rows_host, rows_dev, n_tuner, rcnt.p, QueueArgs(), look.p));
      {
        cudaStream_t st = ctx->stream;
        DBuf<kareto_config> dm;
        DBuf<uint32_t> dmrep, dmout;
        DBuf<uint64_t> dUg;
        std::vector<uint64_t> hUg((size_t)tr->K + 1);
        for (int g = 0; g <= tr->K; g++) hUg[(size_t)g] = (uint64_t)tr->U_g[(size_t)g];
        KTRY(dm.alloc(ctx, mcfg.size())); KTRY(dmrep.alloc(ctx, mrep.size())); KTRY(dmout.alloc(ctx, mout.size()));
        KTRY(dUg.alloc(ctx, hUg.size()));
        KCUDA(ctx, cudaMemcpyAsync(dm.p, mcfg.data(), sizeof(kareto_config) * mcfg.size(), cudaMemcpyHostToDevice, st));
        KCUDA(ctx, cudaMemcpyAsync(dmrep.p, mrep.data(), 4 * mrep.size(), cudaMemcpyHostToDevice, st));
        KCUDA(ctx, cudaMemcpyAsync(dmout.p, mout.data(), 4 * mout.size(), cudaMemcpyHostToDevice, st));
        KCUDA(ctx, cudaMemcpyAsync(dUg.p, hUg.data(), 8 * hUg.size(), cudaMemcpyHostToDevice, st));
        ReplayTrace T{(uint32_t)tr->R, (uint32_t)tr->U, tr->s, tr->arr_rel, tr->grp, tr->blk, tr->inlen, tr->outlen,
                      tr->delta, dUg.p, Nn};
        Pass ps(ctx, "K6_ttl_members", 1, 1);
        k_ttl_member_counts<<<grid_for((int64_t)mcfg.size(), 64), 64, 0, st>>>(
            T, dm.p, dmrep.p, dmout.p, (int64_t)mcfg.size(), look.p, (uint32_t)nrep, rcnt.p, rows_dev, n_tuner, tr->K + 1,
            counts_dev);
        KTRY(sync(ctx, "ttl members"));  // the host vectors above are the copies' sources
      }
      if (!rest.empty()) {
        DBuf<kareto_counts> rc;
        DBuf<uint32_t> drout;
        KTRY(rc.alloc(ctx, rest.size()));
        KTRY(replay_eval(ctx, tr, rest.data(), (int64_t)rest.size(), rows_host, rows_dev, n_tuner, rc.p, QueueArgs(),
                         nullptr));
        KTRY(drout.alloc(ctx, rout.size()));
        KCUDA(ctx, cudaMemcpyAsync(drout.p, rout.data(), 4 * rout.size(), cudaMemcpyHostToDevice, ctx->stream));
        k_scatter_counts<<<grid_for((int64_t)rest.size(), 256), 256, 0, ctx->stream>>>(rc.p, drout.p,
                                                                                       (int64_t)rest.size(), counts_dev);
        KTRY(sync(ctx, "replay scatter"));
      }
      return KARETO_OK;
    }
  }
  // sequence numbers are 32-bit (the LFU key packs (freq << 32 | seq)): one per touch plus one per
  // demotion into a lower tier, and a block entering HBM is demoted at most twice before it is
  // dropped, so seq <= 3N
  if ((uint64_t)tr->N * 3 > 0xFFFFFFFFull)
    return fail(ctx, KARETO_E_OVERFLOW, "replay: %lld accesses exceed the 32-bit sequence range (3N < 2^32)",
                (long long)tr->N);
  KTRY(replay_prepare(ctx, tr));
  cudaStream_t st = ctx->stream;
  const uint64_t U = tr->U > 0 ? (uint64_t)tr->U : 1;
  const int G = tr->K + 1;
  DBuf<uint64_t> dUg;
  {
    std::vector<uint64_t> hUg(G);
    for (int g = 0; g < G; g++) hUg[g] = (uint64_t)tr->U_g[g];
    KTRY(dUg.alloc(ctx, G));
    KCUDA(ctx, cudaMemcpyAsync(dUg.p, hUg.data(), 8 * (size_t)G, cudaMemcpyHostToDevice, st));
    KCUDA(ctx, cudaStreamSynchronize(st));  // hUg is a host temporary
  }
  ReplayTrace T{(uint32_t)tr->R, (uint32_t)tr->U, tr->s, tr->arr_rel, tr->grp, tr->blk, tr->inlen, tr->outlen,
                tr->delta, dUg.p, (uint64_t)tr->N};
  const bool Qm = qarg.model != nullptr;
  const int64_t R = tr->R;
  // classes {list, LFU} x {expiry heap or not}; within a class, neighbours in a warp get
  // similar configurations (policy, TTL row, capacities) so their branches agree more often
  // classes: 0 list, 1 list + expiry heap (FIFO), 2 LFU, 3 LFU + expiry heap, 4 LRU + group lists
  std::vector<uint32_t> cls[5];
  for (int64_t i = 0; i < n; i++) {
    const kareto_config &c = cfg_host[i];
    const uint32_t *tau = rows_host + (size_t)(n_tuner > 0 ? c.tuner : 0) * G;
    bool any_finite = false;
    for (int g = 0; g < G; g++) any_finite |= tau[g] != KARETO_TTL_INF;
    const bool exp = c.cap[2] != KARETO_INF && any_finite;
    const int k = (exp && c.policy == KARETO_LRU) ? 4 : (c.policy == KARETO_LFU ? 2 : 0) + (exp ? 1 : 0);
    cls[k].push_back((uint32_t)i);
  }
  DBuf<kareto_config> dcfg;
  KTRY(dcfg.alloc(ctx, n));
  KCUDA(ctx, cudaMemcpyAsync(dcfg.p, cfg_host, sizeof(kareto_config) * n, cudaMemcpyHostToDevice, st));
  // FIFO / LFU expiry wheel: buckets of 2^BSH ms over [0, span], at most max(256, U/4) of them (so
  // the heads cost <= 1 B per block and configuration)
  const uint32_t a_last = (uint32_t)tr->span_ms;
  uint32_t BSH = 0;
  while (((uint64_t)(a_last >> BSH) + 1) > std::max<uint64_t>(256, U / 4)) BSH++;
  const uint64_t NBK = (uint64_t)(a_last >> BSH) + 1;
  // Concurrent classes (no f3 queue): a wave is one pass over the trace whatever its width (the
  // kernel is latency-bound at these occupancies), so sequential classes waste the unused part
  // of each class's last wave.  Instead every class runs its waves on its own stream with a share
  // of the memory budget proportional to its work (configurations x bytes x relative pass cost),
  // so the classes finish together.
  if (!Qm && getenv("KARETO_K6_SEQUENTIAL") == nullptr) {
    int nonempty = 0;
    for (int q = 0; q < 5; q++) nonempty += !cls[q].empty();
    if (nonempty >= 2) {
      const uint64_t FM = (uint64_t)tr->R + 2;
      const uint64_t NW = (FM + 63) / 64, NSW = (NW + 63) / 64;
      auto per_cfg_of = [&](int q) {
        const bool lfu = q == 2 || q == 3, eheap = q == 1 || q == 3, glist = q == 4;
        return U * (1 + 8) + (eheap || glist ? U * (4 + 8) : 0) + (lfu ? U * 4 + 3 * 8 * (FM + NW + NSW) : 0) +
               (eheap ? 4 * NBK : 0) + (glist ? 8 * (uint64_t)G : 0);
      };
      // relative time of one pass over the trace per class, measured on the config-3 twin (seconds
      // per wave, KARETO_DEBUG, round 2: list 1.85, FIFO + expiry wheel 4.1, LFU 3.6, LFU + expiry
      // wheel 5.95, LRU + group lists 4.2)
      const double pass_cost[5] = {1.0, 2.2, 1.95, 3.2, 2.27};
      double budget = 0;
      KTRY(wave_budget(ctx, 0.8, &budget));
      // every non-empty class first gets one configuration's footprint (so no class is starved
      // to a zero-width wave), the rest of the budget goes in proportion to the classes' work;
      // if even the minimum footprints do not fit, the classes run one after another below
      double wsum = 0, minfoot = 0;
      for (int q = 0; q < 5; q++) {
        wsum += (double)cls[q].size() * (double)per_cfg_of(q) * pass_cost[q];
        if (!cls[q].empty()) minfoot += (double)per_cfg_of(q);
      }
      if (minfoot <= budget) {
      struct ClassState {
        DBuf<uint8_t> tier;
        DBuf<uint32_t> lt, freq, bht, ebh, didx, eht;
        DBuf<uint2> link, elink;
        DBuf<uint64_t> occ;
        RState v{};
        uint64_t W = 0;
        cudaStream_t s = nullptr;
        cudaEvent_t done = nullptr;
      };
      ClassState C[5];
      int launches = 0;
      for (int q = 0; q < 5; q++) {
        std::vector<uint32_t> &ix = cls[q];
        if (ix.empty()) continue;
        std::stable_sort(ix.begin(), ix.end(), [&](uint32_t a, uint32_t b) {
          const kareto_config &x = cfg_host[a], &y = cfg_host[b];
          if (x.policy != y.policy) return x.policy < y.policy;
          if (x.tuner != y.tuner) return x.tuner < y.tuner;
          for (int t = 0; t < 3; t++)
            if (x.cap[t] != y.cap[t]) return x.cap[t] < y.cap[t];
          return false;
        });
        const bool lfu = q == 2 || q == 3, eheap = q == 1 || q == 3, glist = q == 4;
        const uint64_t pc = per_cfg_of(q);
        const double share = (budget - minfoot) * ((double)ix.size() * (double)pc * pass_cost[q]) / wsum;
        uint64_t W = 1 + (uint64_t)(share / (double)pc);
        if (W > ix.size()) W = ix.size();
        if (W > (1u << 20)) W = 1u << 20;
        const uint64_t nwaves = (ix.size() + W - 1) / W;
        W = (ix.size() + nwaves - 1) / nwaves;
        launches += (int)nwaves;
        ClassState &c = C[q];
        c.W = W;
        KTRY(c.tier.alloc(ctx, U * W)); KTRY(c.link.alloc(ctx, U * W));
        if (eheap || glist) KTRY(c.lt.alloc(ctx, U * W));
        if (lfu) {
          KTRY(c.freq.alloc(ctx, U * W)); KTRY(c.bht.alloc(ctx, 6 * FM * W)); KTRY(c.occ.alloc(ctx, 3 * (NW + NSW) * W));
        }
        if (eheap || glist) KTRY(c.elink.alloc(ctx, U * W));
        if (eheap) KTRY(c.ebh.alloc(ctx, NBK * W));
        if (glist) KTRY(c.eht.alloc(ctx, 2 * (size_t)G * W));
        KTRY(c.didx.alloc(ctx, ix.size()));
        KCUDA(ctx, cudaMemcpyAsync(c.didx.p, ix.data(), 4 * ix.size(), cudaMemcpyHostToDevice, st));
        RState &v = c.v;
        v.tier = c.tier.p; v.lt = c.lt.p; v.link = c.link.p;
        if (lfu) {
          v.freq = c.freq.p;
          for (int t = 0; t < 3; t++) {
            v.bh[t] = c.bht.p + (size_t)(2 * t) * FM * W;
            v.bt[t] = c.bht.p + (size_t)(2 * t + 1) * FM * W;
            v.occ[t] = c.occ.p + (size_t)t * (NW + NSW) * W;
            v.occ2[t] = v.occ[t] + NW * W;
          }
          v.NW = (uint32_t)NW;
          v.NSW = (uint32_t)NSW;
        }
        v.ebh = c.ebh.p; v.NB = (uint32_t)NBK; v.BSH = BSH; v.a_last = a_last;
        v.look = look_dev;
        v.look_stride = (uint64_t)n;
        v.elink = c.elink.p;
        v.eh = c.eht.p;
        v.et = c.eht.p + (size_t)G * W;
        v.gblk = tr->gblk;
        v.W = W;
      }
      cudaEvent_t fork;
      const bool dbg = getenv("KARETO_DEBUG") != nullptr;  // per-class finish times
      KCUDA(ctx, cudaEventCreateWithFlags(&fork, dbg ? cudaEventDefault : cudaEventDisableTiming));
      kareto_status rs = KARETO_OK;
      {
        Pass ps(ctx, "K6_replay", 1, launches);
        cudaError_t e = cudaEventRecord(fork, st);  // allocations and index uploads done on st
        QueueKernelArgs qa{};
        for (int q = 0; q < 5 && e == cudaSuccess; q++) {
          const std::vector<uint32_t> &ix = cls[q];
          if (ix.empty()) continue;
          ClassState &c = C[q];
          const bool lfu = q == 2 || q == 3, eheap = q == 1 || q == 3, glist = q == 4;
          const uint64_t W = c.W;
          if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking);
          if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.done, dbg ? cudaEventDefault : cudaEventDisableTiming);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s, fork, 0);
          for (uint64_t w0 = 0; w0 < ix.size() && e == cudaSuccess; w0 += W) {
            const int64_t nw = (int64_t)(ix.size() - w0 < W ? ix.size() - w0 : W);
            cudaMemsetAsync(c.tier.p, 0, U * W, c.s);
            if (eheap || glist) cudaMemsetAsync(c.lt.p, 0xFF, 4 * U * W, c.s);
            if (lfu) {
              cudaMemsetAsync(c.bht.p, 0xFF, 4 * 6 * FM * W, c.s);
              cudaMemsetAsync(c.occ.p, 0, 8 * 3 * (NW + NSW) * W, c.s);
            }
            if (eheap) cudaMemsetAsync(c.ebh.p, 0xFF, 4 * NBK * W, c.s);
            if (glist) cudaMemsetAsync(c.eht.p, 0xFF, 4 * 2 * (size_t)G * W, c.s);
            const unsigned grid = (unsigned)((nw + 63) / 64);
            const uint32_t *wi = c.didx.p + w0;
#define KREPC(L, E) k_replay<L, E, false><<<grid, 64, 0, c.s>>>(T, dcfg.p, wi, rows_dev, n_tuner, G, c.v, nw, counts_dev, qa)
            if (q == 0) KREPC(false, 0);
            if (q == 1) KREPC(false, 1);
            if (q == 2) KREPC(true, 0);
            if (q == 3) KREPC(true, 1);
            if (q == 4) KREPC(false, 2);
#undef KREPC
            e = cudaGetLastError();
          }
        }
        // join every started class before the buffers are freed on st (also on errors)
        for (int q = 0; q < 5; q++) {
          if (!C[q].s) continue;
          if (C[q].done && cudaEventRecord(C[q].done, C[q].s) == cudaSuccess) cudaStreamWaitEvent(st, C[q].done, 0);
          else cudaStreamSynchronize(C[q].s);
        }
        if (e != cudaSuccess) rs = fail(ctx, KARETO_E_CUDA, "concurrent replay: %s", cudaGetErrorString(e));
      }
      if (rs == KARETO_OK) rs = sync(ctx, "replay");
      else cudaStreamSynchronize(st);
      if (dbg && rs == KARETO_OK)
        for (int q = 0; q < 5; q++) {
          float ms = 0.f;
          if (C[q].done && cudaEventElapsedTime(&ms, fork, C[q].done) == cudaSuccess)
            fprintf(stderr, "[kareto] K6 class %d: %zu configs, waves of %llu, done after %.1f ms\n", q,
                    cls[q].size(), (unsigned long long)C[q].W, ms);
        }
      for (int q = 0; q < 5; q++) {
        if (C[q].s) cudaStreamDestroy(C[q].s);
        if (C[q].done) cudaEventDestroy(C[q].done);
      }
      cudaEventDestroy(fork);
      pool_trim(ctx);
      return rs;
      }
    }
  }
  for (int q = 0; q < 5; q++) {
    std::vector<uint32_t> &ix = cls[q];
    if (ix.empty()) continue;
    const bool lfu = q == 2 || q == 3, eheap = q == 1 || q == 3, glist = q == 4;
    std::stable_sort(ix.begin(), ix.end(), [&](uint32_t a, uint32_t b) {
      const kareto_config &x = cfg_host[a], &y = cfg_host[b];
      if (x.policy != y.policy) return x.policy < y.policy;
      if (x.tuner != y.tuner) return x.tuner < y.tuner;
      for (int t = 0; t < 3; t++)
        if (x.cap[t] != y.cap[t]) return x.cap[t] < y.cap[t];
      return false;
    });
    // LFU frequency buckets: a resident block's frequency is at most its accesses (<= R)
    const uint64_t FM = (uint64_t)tr->R + 2;
    const uint64_t NW = (FM + 63) / 64, NSW = (NW + 63) / 64;
    uint64_t per_cfg = U * (1 + 8) + (eheap || glist ? U * (4 + 8) : 0) + (lfu ? U * 4 + 3 * 8 * (FM + NW + NSW) : 0) +
                       (eheap ? 4 * NBK : 0) + (glist ? 8 * (uint64_t)G : 0);
    if (Qm) per_cfg += 16 * (uint64_t)R + 8 * (uint64_t)qarg.model->instances + 64;  // f3: TTFT rows + queue
    // 80% of free device memory per wave (60% left the LRU expiry-list class of the config-3 twin
    // in two waves, i.e. two passes over the trace: 7.1 s -> 4.7 s at 80%)
    double budget = 0;
    KTRY(wave_budget(ctx, 0.8, &budget));
    uint64_t W = (uint64_t)budget / per_cfg;
    if (W > (1u << 20)) W = 1u << 20;
    if (W > ix.size()) W = ix.size();
    if (W < 1) return fail(ctx, KARETO_E_OOM, "replay needs %llu bytes per configuration", (unsigned long long)per_cfg);
    // balance the waves
    const uint64_t nwaves = (ix.size() + W - 1) / W;
    W = (ix.size() + nwaves - 1) / nwaves;
    DBuf<uint8_t> tier;
    DBuf<uint32_t> lt, freq, bht, ebh, didx;
    DBuf<uint2> link, elink;
    DBuf<uint64_t> occ;
    DBuf<uint32_t> eht;
    KTRY(tier.alloc(ctx, U * W)); KTRY(link.alloc(ctx, U * W));
    if (eheap || glist) KTRY(lt.alloc(ctx, U * W));
    if (lfu) {
      KTRY(freq.alloc(ctx, U * W)); KTRY(bht.alloc(ctx, 6 * FM * W)); KTRY(occ.alloc(ctx, 3 * (NW + NSW) * W));
    }
    if (eheap || glist) KTRY(elink.alloc(ctx, U * W));
    if (eheap) KTRY(ebh.alloc(ctx, NBK * W));
    if (glist) KTRY(eht.alloc(ctx, 2 * (size_t)G * W));
    KTRY(didx.alloc(ctx, ix.size()));
    KCUDA(ctx, cudaMemcpyAsync(didx.p, ix.data(), 4 * ix.size(), cudaMemcpyHostToDevice, st));
    RState v{};
    v.tier = tier.p; v.lt = lt.p; v.link = link.p;
    if (lfu) {
      v.freq = freq.p;
      for (int t = 0; t < 3; t++) {
        v.bh[t] = bht.p + (size_t)(2 * t) * FM * W;
        v.bt[t] = bht.p + (size_t)(2 * t + 1) * FM * W;
        v.occ[t] = occ.p + (size_t)t * (NW + NSW) * W;
        v.occ2[t] = v.occ[t] + NW * W;
      }
      v.NW = (uint32_t)NW;
      v.NSW = (uint32_t)NSW;
    }
    v.ebh = ebh.p; v.NB = (uint32_t)NBK; v.BSH = BSH; v.a_last = a_last;
    v.look = look_dev;
    v.look_stride = (uint64_t)n;
    v.elink = elink.p;
    v.eh = eht.p;
    v.et = eht.p + (size_t)G * W;
    v.gblk = tr->gblk;
    v.W = W;
    QueueKernelArgs qa{};
    DBuf<double> qF, qt, qts;
    DBuf<int64_t> qoff;
    DBuf<uint8_t> qtmp;
    if (Qm) {
      qa.m = *qarg.model;
      KTRY(qF.alloc(ctx, (size_t)qarg.model->instances * W)); KTRY(qt.alloc(ctx, (size_t)W * R));
      KTRY(qts.alloc(ctx, (size_t)W * R)); KTRY(qoff.alloc(ctx, W + 1));
      qa.F = qF.p; qa.ttft = qt.p; qa.out = qarg.out_dev; qa.span_ms = qarg.span_ms; qa.LO = qarg.LO;
    }
    for (uint64_t w0 = 0; w0 < ix.size(); w0 += W) {
      const int64_t nw = (int64_t)(ix.size() - w0 < W ? ix.size() - w0 : W);
      KCUDA(ctx, cudaMemsetAsync(tier.p, 0, U * W, st));
      if (eheap || glist) KCUDA(ctx, cudaMemsetAsync(lt.p, 0xFF, 4 * U * W, st));
      if (lfu) {
        KCUDA(ctx, cudaMemsetAsync(bht.p, 0xFF, 4 * 6 * FM * W, st));
        KCUDA(ctx, cudaMemsetAsync(occ.p, 0, 8 * 3 * (NW + NSW) * W, st));
      }
      if (eheap) KCUDA(ctx, cudaMemsetAsync(ebh.p, 0xFF, 4 * NBK * W, st));
      if (glist) KCUDA(ctx, cudaMemsetAsync(eht.p, 0xFF, 4 * 2 * (size_t)G * W, st));
      static const char *kPassName[5] = {"K6_replay_list", "K6_replay_list_exp", "K6_replay_lfu", "K6_replay_lfu_exp",
                                         "K6_replay_lru_exp"};
      Pass ps(ctx, kPassName[q], 1, 1);
      const unsigned grid = (unsigned)((nw + 63) / 64);
      const uint32_t *wi = didx.p + w0;
#define KREP(L, E, QQ) k_replay<L, E, QQ><<<grid, 64, 0, st>>>(T, dcfg.p, wi, rows_dev, n_tuner, G, v, nw, counts_dev, qa)
      if (!Qm) {
        if (q == 0) KREP(false, 0, false);
        if (q == 1) KREP(false, 1, false);
        if (q == 2) KREP(true, 0, false);
        if (q == 3) KREP(true, 1, false);
        if (q == 4) KREP(false, 2, false);
      } else {
        if (q == 0) KREP(false, 0, true);
        if (q == 1) KREP(false, 1, true);
        if (q == 2) KREP(true, 0, true);
        if (q == 3) KREP(true, 1, true);
        if (q == 4) KREP(false, 2, true);
      }
#undef KREP
      if (Qm && R > 0) {  // exact nearest-rank P99 of each configuration's TTFT row (R53)
        Pass pq(ctx, "F3_p99", 1, 2);
        k_row_offsets<<<grid_for(nw + 1, 256), 256, 0, st>>>(nw, R, qoff.p);
        size_t bytes = 0;
        KCUDA(ctx, cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, qt.p, qts.p, nw * R, nw, qoff.p, qoff.p + 1, st));
        if (bytes > qtmp.n) KTRY(qtmp.alloc(ctx, bytes));
        bytes = qtmp.n;
        KCUDA(ctx, cub::DeviceSegmentedSort::SortKeys(qtmp.p, bytes, qt.p, qts.p, nw * R, nw, qoff.p, qoff.p + 1, st));
        k_pick_p99_idx<<<grid_for(nw, 256), 256, 0, st>>>(qts.p, R, nw, (99 * R + 99) / 100, wi, qarg.out_dev);
      }
    }
    KTRY(sync(ctx, "replay"));
  }
  pool_trim(ctx);
  return KARETO_OK;
}

}  // namespace kareto

// trace_load.cuh -- host-level building blocks of trace loading, shared by the whole-trace
// load (trace_load.cu) and the time-sharded load (trace_shard.cu).  Not part of the ABI.
#pragma once

#include "internal.cuh"

namespace kareto {

enum : uint32_t { F_OFFSETS = 1, F_OUTPUT = 2, F_INPUT_LEN = 4, F_CHAIN = 8, F_DELTA = 16 };

struct LoadStats {  // device-side accumulators, copied back once
  unsigned long long sl_lo, sl_hi, sq_lo, sq_hi, O;
  unsigned long long n_total;
  unsigned int flags, max_blocks;
  long long arr_first, arr_last;
};

// State of row a1 (ingest) kept for the later steps.
struct Ingest {
  DBuf<int64_t> h_arr, h_off, h_in;
  DBuf<int32_t> h_out;
  const int64_t *arrival = nullptr, *offsets = nullptr, *input_tokens = nullptr;
  const int32_t *out_tok = nullptr;
  int64_t total = 0;        // offsets[R]: elements of tokens / block_hash
  DBuf<int64_t> src_off;    // [R] sorted request -> offset of its tokens / hashes
  DBuf<uint64_t> nblk;      // [R+1] blocks per sorted request
  DBuf<LoadStats> stats;
  LoadStats hs{};
};

// a1: validate, stable-sort requests by (arrival, index), per-request metadata, block
// starts.  Fills tr->{R, K, arr, s, inlen, outlen, N, max_blocks, span_ms, O, SL, SQ, Ltok}.
kareto_status ingest(kareto_ctx *ctx, const kareto_trace_desc *d, kareto_trace *tr, Ingest &in);

// The token (TOKENS) or hash (HASHES) elements [lo, hi) on the device.  *base is shifted so
// that base[i] is element i for i in [lo, hi) (no copy when the inputs are on the device).
kareto_status upload_payload(kareto_ctx *ctx, const kareto_trace_desc *d, int64_t lo, int64_t hi,
                             DBuf<uint32_t> &tok, DBuf<uint64_t> &bh, const uint32_t **tok_base,
                             const uint64_t **bh_base);

// qf[i] = 1 if sorted element i is the first occurrence of its hash in the range, nx[i] = 1 if
// a later occurrence exists (both in sorted order, produced by the link kernels).
struct SortedHashes {
  DBuf<uint32_t> key;
  DBuf<uint64_t> val;
  DBuf<uint8_t> qf, nx;
};

// a2 (K1) over the sorted requests [r0, r1) whose blocks occupy global positions [P0, P1)
// (tok_base[i] valid for i < tok_end):
// hash_out / req_out are indexed by (position - P0); req_out holds global request indices.
kareto_status chain_hash(kareto_ctx *ctx, const kareto_trace_desc *d, const kareto_trace *tr, const Ingest &in,
                         const uint32_t *tok_base, const uint64_t *bh_base, int64_t tok_end, int64_t r0, int64_t r1,
                         uint64_t *hash_out, uint32_t *req_out, SortedHashes *prep);

// a3 (K2 link): prev[i] = largest i' < i with hash[i'] == hash[i] (local indices), kNone if
// none.  With keep != nullptr the fingerprint-sorted (key, value) arrays are handed back:
// key = top 32 bits of m = fmix64(h ^ C), value = (low 32 bits of m) << 32 | i.
// prep: K2's sort input already written by K1 (chain_hash with prep), or nullptr / empty
kareto_status link_prev(kareto_ctx *ctx, const uint64_t *hash, uint64_t n, uint32_t *prev, SortedHashes *keep,
                        SortedHashes *prep = nullptr, unsigned *bucket_ovf = nullptr);

// The bijective mix whose halves are the sort key / value high word (k_sort_prep).
constexpr uint64_t kSortMixC = 0x6A09E667F3BCC909ULL;

// K3 run list: heads compacted from the flags (start), then per run request / length / first
// previous position once the host knows M (finish); stack_depth_runs runs K3 proper on it.
struct RunList {
  DBuf<uint32_t> run_start, run_req, run_len, run_p0;
  DBuf<int> m_dev;
  int M = 0;
};
kareto_status run_list_start(kareto_ctx *ctx, uint64_t N, const uint8_t *run_flag, RunList &rl);
kareto_status run_list_finish(kareto_ctx *ctx, uint64_t N, const uint32_t *prev_c, const uint32_t *req,
                              uint32_t req_base, const uint32_t *s, uint32_t pos_base, int M, RunList &rl);
kareto_status stack_depth_runs(kareto_ctx *ctx, uint64_t N, uint64_t y_range, const uint32_t *s,
                               uint32_t pos_base, uint32_t y_off, RunList &rl, uint32_t *depth, int64_t *n_runs,
                               uint4 **runs_out = nullptr);
kareto_status stack_depth(kareto_ctx *ctx, uint64_t n, uint64_t y_range, const uint32_t *prev_c,
                          const uint32_t *req, uint32_t req_base, const uint32_t *s, uint32_t pos_base,
                          uint32_t y_off, const uint8_t *run_flag, uint32_t *depth, int64_t *n_runs,
                          uint4 **runs_out = nullptr);

}  // namespace kareto

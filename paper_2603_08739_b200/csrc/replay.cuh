// replay.cuh -- K6 per-configuration replay (replay.cu), used by eval.cu.
#pragma once
#include <cub/cub.cuh>

#include "internal.cuh"

namespace kareto {

struct ReplayTrace {
  uint32_t R, U;
  const uint32_t *s;       // [R+1] first touch position of each request
  const uint32_t *arr;     // [R] arrival ms relative to the first request
  const uint16_t *grp;     // [R] group of each request
  const uint32_t *blk;     // [N] dense block id of each access (touch order)
  const uint32_t *inlen;   // [R] input tokens (row f3 queue)
  const uint32_t *outlen;  // [R] output tokens (row f3 queue)
  const uint32_t *delta;   // [N] reuse interval of each access (kNone: first access), touch order
  const uint64_t *Ug;      // [K+1] distinct blocks per group
  uint64_t N;              // accesses
};

// row f3 (queue.cu): the queue model evaluated inside the replay of each configuration
struct QueueArgs {
  const kareto_model *model = nullptr;  // host; null = no queue
  kareto_queue_result *out_dev = nullptr;  // [n] in the caller's configuration order
  uint64_t span_ms = 0, LO = 0;
};

// dense block ids / groups / relative arrivals (lazily, cached in the trace)
kareto_status replay_prepare(kareto_ctx *ctx, kareto_trace *tr);
// counts of n configurations (host array) into counts_dev[n]; rows = [max(n_tuner,1)][K+1]
// TTL rows, on the host and on the device
// look_dev (optional, [n][N] bytes): each configuration's lookup tiers (HBM / DRAM / none) per access
kareto_status replay_eval(kareto_ctx *ctx, kareto_trace *tr, const kareto_config *cfg_host, int64_t n,
                          const uint32_t *rows_host, const uint32_t *rows_dev, int n_tuner,
                          kareto_counts *counts_dev, const QueueArgs &q = QueueArgs(), uint8_t *look_dev = nullptr);

}  // namespace kareto

/*
 * kareto.h -- C ABI of the B200-native Kareto configuration-evaluation hot path.
 *
 * Kareto (arXiv 2603.08739) searches tiered KV-cache storage configurations: a planner
 * proposes configurations (DRAM capacity, disk TTL, disk medium; PAPER.md 4.1 line 506),
 * a simulator replays "request arrival times, input/output token lengths, and
 * token-level KV-block hashes" against each and a selector keeps the
 * non-dominated ones (Alg. 1 line 22 "ParetoFilter(P)").  This library
 * evaluates very many configurations against one trace on the GPU:
 *
 *   kareto_load_trace  -- ingest, chained 16-token block hashes ("salted hash
 *                         blocks (16 tokens per block)"), previous access / reuse
 *                         interval / prefix-subtree group of every block access
 *                         (P:601), exact LRU stack depths.
 *   kareto_eval_grid   -- per-configuration tier hit/miss/eviction counts and the
 *                         objective vector of Eq. 1 with the cost of Eq. 2
 *                         (P:227-231), for many configurations at once.
 *   kareto_pareto      -- diminishing-return pruning (Alg. 1 expansion test,
 *                         P:555-559) then non-dominance.
 *
 * Readings of the paper (R1..R35) and the exact semantics are in DESIGN.md.
 *
 * Conventions
 *   - Every function returns a kareto_status; no exception crosses the ABI.  On failure a
 *     message is available from kareto_last_error(ctx) until the next call on that ctx.
 *   - Ownership: the caller owns every buffer it passes.  Trace inputs are copied at load;
 *     handles (kareto_ctx, kareto_trace) are owned by the library and released with
 *     kareto_destroy / kareto_trace_free.
 *   - Synchronicity: every call returns after its work on the context stream is complete.
 *   - Device pointers must be cudaMalloc'd (or cudaMallocAsync'd) memory of the context
 *     device; host pointers are ordinary (pinned memory makes copies faster).
 *   - Multi-GPU: with world > 1 every rank calls kareto_eval_grid collectively with the
 *     FULL identical configuration list; each evaluates a deterministic shard and the
 *     objective vectors and counts are all-gathered over NCCL (NVLink), so outputs are
 *     complete and byte-identical on every rank.
 */
#ifndef KARETO_H
#define KARETO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KARETO_OK = 0,
  KARETO_E_INVALID = 1,     /* bad argument / configuration / model constant          */
  KARETO_E_PARSE = 2,       /* malformed trace arrays (offsets decreasing, ...)       */
  KARETO_E_CHAIN = 3,       /* block hashes are not chain-consistent (R7)   */
  KARETO_E_OOM = 4,         /* device memory exhausted                                */
  KARETO_E_CUDA = 5,        /* CUDA runtime error                                     */
  KARETO_E_NCCL = 6,        /* NCCL error (world > 1)                                 */
  KARETO_E_OVERFLOW = 7,    /* a 32/64-bit bound of the data layout is exceeded       */
  KARETO_E_UNSUPPORTED = 8  /* valid request this build cannot evaluate               */
} kareto_status;

typedef struct kareto_ctx kareto_ctx;     /* device, borrowed stream, arena, NCCL comm */
typedef struct kareto_trace kareto_trace; /* device-resident, immutable after load      */

/* Create a context on CUDA `device`, enqueueing all work on `cuda_stream` (a cudaStream_t;
 * NULL = legacy default stream; borrowed, not destroyed).  For world > 1 pass the 128-byte
 * NCCL unique id produced on rank 0 by kareto_nccl_unique_id() and broadcast by the
 * caller; for world == 1 pass NULL -- or an id, which creates a 1-rank NCCL communicator so
 * that every collective (the eval_grid allgather, the time-sharded load's all-to-all and
 * allreduces) runs through NCCL on one GPU.  Errors: KARETO_E_INVALID (rank/world), _E_CUDA,
 * _E_NCCL.
 * Threads: a context, and the traces and grids made with it, are used by one host thread at a
 * time (calls are synchronous on its stream); different contexts may run on different threads. */
kareto_status kareto_create(int device, void *cuda_stream, const void *nccl_unique_id, int rank, int world,
                            kareto_ctx **out);
void kareto_destroy(kareto_ctx *ctx);
/* Message of the last failed call on ctx (per-context buffer; valid until the next call). */
const char *kareto_last_error(const kareto_ctx *ctx);
/* Writes a 128-byte NCCL unique id to out (rank 0, world > 1). KARETO_E_NCCL if NCCL is absent. */
kareto_status kareto_nccl_unique_id(void *out128);

/* In-process rank group ("loopback"): world contexts of ONE process on one device, each driven
 * by its own host thread, exchanging through each other's device buffers instead of NCCL.
 * Every multi-rank path of this library (configuration sharding in kareto_eval_grid, the
 * time-sharded load below) runs unchanged on it, which is how those paths are tested where
 * only one GPU exists.  The group is owned by the caller and must outlive its contexts.
 * Errors: KARETO_E_INVALID (world outside [1, 1024], rank outside [0, world)), _E_CUDA. */
typedef struct kareto_loopback kareto_loopback;
kareto_status kareto_loopback_create(int32_t world, kareto_loopback **out);
void kareto_loopback_destroy(kareto_loopback *group);
int32_t kareto_loopback_world(const kareto_loopback *group);
kareto_status kareto_create_loopback(int device, void *cuda_stream, kareto_loopback *group, int rank,
                                     kareto_ctx **out);

/* ---------------------------------------------------------------- trace ---- */
typedef enum { KARETO_TOKENS = 0, KARETO_HASHES = 1 } kareto_input_mode;

typedef struct {
  int64_t n_requests;           /* R >= 1                                                     */
  const int64_t *arrival_ms;    /* [R] arrival in ms, any order; stable-sorted by (arrival,
                                   index) inside (R6)                               */
  const int32_t *output_tokens; /* [R] >= 0 decode lengths                                    */
  int32_t mode;                 /* kareto_input_mode                                          */
  const int64_t *offsets;       /* [R+1] nondecreasing; TOKENS: token offsets into tokens;
                                   HASHES: block offsets into block_hash                      */
  const uint32_t *tokens;       /* TOKENS: [offsets[R]] input token ids; only full 16-token
                                   blocks are hashed (R1, R3)                                 */
  const uint64_t *block_hash;   /* HASHES: [offsets[R]] chained hashes, one per full block   */
  const int64_t *input_tokens;  /* HASHES: [R] input lengths (>= 16*blocks) or NULL = 16*blocks */
  uint64_t salt;                /* TOKENS: hash salt (R2)                                     */
  int32_t top_k;                /* K >= 0 prefix-subtree groups (+1 residual, R23), K <= 1023  */
  int32_t inputs_on_device;     /* 1: all pointers above are device pointers; 0: host         */
} kareto_trace_desc;

/* Load a trace: sort, hash (TOKENS), per-access previous position / reuse interval /
 * group, LRU stack depth.  Validation errors: KARETO_E_INVALID
 * (R < 1, K out of range, null pointers), _E_PARSE (offsets decreasing, output < 0,
 * input_tokens < 16*blocks), _E_CHAIN (R7), _E_OVERFLOW (>= 2^32-1 block accesses or a
 * reuse interval >= 2^32-1 ms), _E_OOM.
 * Memory: the trace keeps 24 B per access (+ 16 B per K3 run) on the device until
 * kareto_trace_free; two context scratch buffers stay with the context for the next load and
 * are freed by kareto_destroy: the K2 link's (~20 B per access) and, for host inputs
 * (inputs_on_device = 0), the device staging copy of the tokens / block hashes (grown to the
 * largest load). */
kareto_status kareto_load_trace(kareto_ctx *ctx, const kareto_trace_desc *desc, kareto_trace **out);
void kareto_trace_free(kareto_trace *tr);

typedef struct {
  int64_t n_requests, n_accesses, n_unique, span_ms;
  uint64_t input_tokens, output_tokens; /* Ltok = sum L_r, O = sum o_r               */
  int32_t top_k;
  int32_t max_blocks_per_request;
} kareto_trace_info;
/* Scalars, and per-group |B_g| (unique blocks) and N_g (reuse events) [K+1] (
 * either array may be NULL).  Host pointers. */
kareto_status kareto_trace_stats(const kareto_trace *tr, kareto_trace_info *info, int64_t *group_unique,
                                 int64_t *group_reuse);

typedef enum {
  KARETO_X_HASH = 0,    /* uint64 [N] chained hash of each access, touch order         */
  KARETO_X_PREV = 1,    /* uint32 [N] previous position of the same block, UINT32_MAX = none */
  KARETO_X_DELTA = 2,   /* uint32 [N] reuse interval ms, UINT32_MAX = first access      */
  KARETO_X_REQ = 3,     /* uint32 [N] request (sorted index) of each access             */
  KARETO_X_DEPTH = 4,   /* uint32 [N] LRU depth d at request start, UINT32_MAX = first  */
  KARETO_X_GROUP = 5,   /* uint16 [R] group of each request (sorted order)              */
  KARETO_X_START = 6    /* uint32 [R+1] first touch position of each request            */
} kareto_export;
/* Copy one per-access array (touch order: request by request, blocks leaf -> root, R12)
 * to host memory `out`.  Diagnostics / parity testing. */
kareto_status kareto_trace_export(kareto_ctx *ctx, const kareto_trace *tr, int32_t which, void *out);

/* ----------------------------------------------------------- evaluation ---- */
enum { KARETO_LRU = 0, KARETO_FIFO = 1, KARETO_LFU = 2 };
#define KARETO_INF UINT64_MAX   /* cap[2] == KARETO_INF => TTL (lease) mode (R19)           */
#define KARETO_NA UINT64_MAX    /* counts: value not defined for this configuration        */
#define KARETO_TTL_INF UINT32_MAX

typedef struct {
  uint64_t cap[3];   /* HBM, DRAM, disk capacities in 16-token blocks (R14); cap[2] == KARETO_INF
                        selects TTL mode                                                  */
  uint8_t policy;    /* KARETO_LRU / _FIFO / _LFU (R24)                                    */
  uint8_t medium;    /* index into kareto_model.media                                      */
  uint16_t tuner;    /* row of the per-group TTL table (ms) applied to the disk tier (R17) */
  int32_t axis[3];   /* grid coordinates along HBM / DRAM / disk, used by pruning (R34)    */
} kareto_config;     /* 40 bytes */

typedef struct {
  uint64_t hit[3];            /* prefix hits served by HBM, DRAM, disk                     */
  uint64_t miss;              /* block accesses recomputed                                 */
  uint64_t evict[3];          /* HBM->DRAM, out of DRAM, disk capacity drops (NA when a
                                 finite TTL is in force in CAPACITY mode; 0 in TTL mode)   */
  uint64_t disk_writes;       /* DRAM->disk demotions (CAPACITY, c3 > 0) / lease starts (TTL) */
  uint64_t hit_pos_sum;       /* sum of chain positions k over hits                        */
  uint64_t bytetime_block_ms; /* TTL mode: sum_g C_g(tau_g), block*ms              */
  uint64_t resident_after_hole; /* diagnostic: resident blocks after the first miss        */
} kareto_counts;              /* 88 bytes */

typedef struct { double bw_base, bw_slope, bw_max, price; } kareto_medium;
  /* bytes/s, bytes/s per provisioned GB, bytes/s cap, $ per GB-hour     */
typedef struct { double breakpoint, rate, jump; } kareto_phi_segment;
  /* phi_IOPS: usage >= breakpoint adds jump + rate*(min(usage, next) - breakpoint)
     $/IOPS-month, right-continuous (R32)                                 */
typedef struct {
  int32_t instances, gpus_per_instance;   /* I, G                                      */
  uint64_t alpha_ps, beta_ps, dec_ps;     /* prefill ps/token, ps/token/position, decode ps/token */
  uint64_t block_bytes;                   /* Bb: KV bytes per 16-token block           */
  double bw_dram;                         /* bytes/s                                   */
  double c_hw, p_hbm, p_dram;             /* $/GPU-hour, $/GB-hour                     */
  double iops_per_block;                  /* IOPS per block transfer                   */
  double ttl_prov_gb;                     /* TTL mode: provisioned GB for the bandwidth curve */
  int32_t n_media, n_phi;                 /* 1..8, 0..8                                */
  kareto_medium media[8];
  kareto_phi_segment phi[8];
} kareto_model;

/* Evaluate n_cfg configurations (host array) against a loaded trace.
 *   ttl_ms    host [n_tuner][K+1] per-group disk TTLs in ms (KARETO_TTL_INF = infinity);
 *             NULL with n_tuner == 0 means every tuner index reads an all-infinite row.
 *   counts_out [n_cfg] or NULL; obj_out [n_cfg][3] = (mean TTFT ms, -tokens/s, cost $) or NULL;
 *   outputs_on_device selects device (1) or host (0) output pointers.
 * Errors: KARETO_E_INVALID (policy > 2, tuner >= n_tuner, medium >= n_media, TTL mode with
 * an infinite TTL (R22), invalid model constants), _E_UNSUPPORTED (a configuration needs
 * the per-configuration replay and this build has none for it), _E_OVERFLOW (also: replay
 * configurations on a trace with 3N >= 2^32 accesses, the K6 sequence range), _E_OOM (one
 * replay configuration's state does not fit the device), _E_NCCL.
 * Memory: K6 replay state is sized per wave to 80% of the free device memory (divided among
 * loopback ranks sharing the GPU; env KARETO_K6_BUDGET=<bytes> overrides) and returned to the
 * device after the call (the stream-ordered pool is trimmed). */
kareto_status kareto_eval_grid(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg, int64_t n_cfg,
                               const uint32_t *ttl_ms, int32_t n_tuner, const kareto_model *model,
                               kareto_counts *counts_out, double *obj_out, int32_t outputs_on_device);

typedef struct {
  int32_t enabled; /* 0: no pruning                                                      */
  double tau_e;    /* relative latency-gain threshold (default 0.05, R34)               */
} kareto_prune;
/* Select: status_out[i] = 2 pruned (R34), 1 frontier, 0 dominated (R35).  obj and
 * status_out are device (on_device = 1) or host (0) pointers; cfg is a host array (its
 * axis / policy / medium / tuner define the pruning lines; when pruning is enabled axis
 * values must lie in [0, 65536) and tuner < 1024, else KARETO_E_INVALID).  n_frontier
 * (host, may be NULL) receives the number of frontier configurations. */
kareto_status kareto_pareto(kareto_ctx *ctx, const double *obj, const kareto_config *cfg, int64_t n,
                            const kareto_prune *prune, uint8_t *status_out, int64_t *n_frontier,
                            int32_t on_device);

/* ------------------------------------------------- prepared grids ---- */
/* A configuration grid prepared once for repeated evaluation -- Alg. 1's rounds, one trace per
 * time window ("historical traces from a recent time window"), bench steps: the host work
 * of kareto_eval_grid / kareto_pareto that depends on the configurations and the TTL table only
 * (validation of every configuration, the rank's cost-weighted shard, the stack-path / replay
 * split, the TTL value sets, the line-key widths of pruning) and the device copies they need.
 * It also keeps, from its first use, what depends on the grid and the trace's U only: K4's sorted
 * boundary set, its lookup table and the per-configuration indices (recomputed when a trace with
 * another U is evaluated), and K8a's sorted line order per axis (~12 B per configuration and
 * axis) -- a step then runs only the per-trace passes.
 *   cfg [n_cfg], ttl_ms [n_tuner][n_groups] host, as for kareto_eval_grid (n_groups = K+1 of the
 *   traces it will be evaluated on; eval returns KARETO_E_INVALID for another K).
 * The grid copies everything it keeps; the caller's arrays may be reused at once.  It belongs to
 * `ctx` (its device memory lives on the context's stream): free it with kareto_grid_free before
 * kareto_destroy.  Model-dependent checks (medium < n_media, capacities x block bytes < 2^64) run
 * at evaluation from stored maxima.  Errors: as kareto_eval_grid's configuration errors, _E_OOM. */
typedef struct kareto_grid kareto_grid;
kareto_status kareto_grid_create(kareto_ctx *ctx, const kareto_config *cfg, int64_t n_cfg, const uint32_t *ttl_ms,
                                 int32_t n_tuner, int32_t n_groups, kareto_grid **out);
void kareto_grid_free(kareto_grid *grid);
/* kareto_eval_grid over a prepared grid (same outputs, bit-identical).  A grid created on a
 * multi-rank context holds its rank's configuration shard; evaluated against a time-sharded
 * trace (every rank evaluates the whole grid) it derives and keeps the unsharded split on first
 * use. */
kareto_status kareto_eval_grid_prepared(kareto_ctx *ctx, const kareto_trace *tr, const kareto_grid *grid,
                                        const kareto_model *model, kareto_counts *counts_out, double *obj_out,
                                        int32_t outputs_on_device);
/* kareto_pareto over a prepared grid's configurations (n = the grid's n_cfg; same outputs).
 * Pruning with line keys out of range returns the KARETO_E_INVALID kareto_pareto would. */
kareto_status kareto_pareto_prepared(kareto_ctx *ctx, const double *obj, const kareto_grid *grid,
                                     const kareto_prune *prune, uint8_t *status_out, int64_t *n_frontier,
                                     int32_t on_device);

/* Host-only helper (no device work): the count-balanced contiguous shard [*lo, *hi) =
 * [floor(n rank / world), floor(n (rank+1) / world)) -- what kareto_shard_bounds returns when
 * every configuration takes the stack path. */
kareto_status kareto_shard_range(int64_t n, int32_t rank, int32_t world, int64_t *lo, int64_t *hi);

/* Host-only helper: the contiguous shards kareto_eval_grid evaluates on `world` ranks,
 * balanced by estimated cost: a stack-path configuration weighs 1, a K6 replay
 * configuration 10^6 x its class's relative trace-pass time.  bounds [world+1] (host):
 * rank r evaluates [bounds[r], bounds[r+1]); unit weights reproduce kareto_shard_range.
 * cfg / ttl_ms host, as passed to kareto_eval_grid; n_groups = K+1 of the trace.
 * Errors: KARETO_E_INVALID (bad sizes, tuner >= n_tuner). */
kareto_status kareto_shard_bounds(const kareto_config *cfg, int64_t n, const uint32_t *ttl_ms, int32_t n_tuner,
                                  int32_t n_groups, int32_t world, int64_t *bounds);

/* ------------------------------------------------------ row f1: search ---- */
/* Exact 3-D hypervolume ("We compute hypervolume using an identical dominated
 * reference point"; R41): the Lebesgue measure of the union of the boxes [obj_i, ref] of the
 * points with mask[i] != 0 (mask NULL: all n), minimisation in all three objectives.
 *   obj   [n][3] device (on_device = 1) or host (0); mask [n] same space or NULL;
 *   ref   host [3]; hv_out host.
 * Errors: KARETO_E_INVALID when some selected point is not strictly better than ref in every
 * objective (the message names its index) or n < 0. */
kareto_status kareto_hypervolume(kareto_ctx *ctx, const double *obj, const uint8_t *mask, int64_t n,
                                 const double ref[3], double *hv_out, int32_t on_device);

/* Alg. 1 "Adaptive Pareto Exploration" over the DRAM-capacity x disk-TTL
 * plane: HBM fixed at hbm_gb; DRAM d GB; TTL (lease) mode with a uniform disk TTL of t seconds
 * for every group; GB -> blocks = floor(GB * 1e9 / block_bytes) (R14).  Each round's
 * candidates are evaluated in one kareto_eval_grid call (sharded over the context's ranks);
 * the expansion / refinement decisions follow DESIGN.md R36-R40. */
typedef struct {
  double hbm_gb;                      /* fixed HBM capacity per instance, GB               */
  int64_t d_min, d_max, d_step;       /* initial DRAM range and step, GB (d_step >= 1)     */
  int64_t t_min, t_max, t_step;       /* initial disk-TTL range and step, s (t_step >= 1)  */
  double tau_e, tau_perf, tau_cost;   /* expand / refine thresholds, relative (R36)        */
  int32_t policy;                     /* KARETO_LRU (stack path) / _FIFO / _LFU (K6)       */
  int32_t max_rounds;                 /* 0 = until no candidates remain                    */
  int32_t expand_ttl;                 /* 0 = Alg. 1 as written (only the DRAM axis expands,
                                         R37); 1 = also the TTL axis, symmetrically at the
                                         lowest DRAM row (R55, an extension)     */
  int32_t pad;
} kareto_search_params;
typedef struct {
  int64_t d_gb, t_s;                  /* the evaluated configuration                       */
  double obj[3];                      /* mean TTFT ms, -tokens/s, cost $                   */
  int32_t round;                      /* evaluation round (0 = the seed grid)              */
  uint8_t status;                     /* 1: on the Pareto frontier of all evaluated points */
  uint8_t pad[3];
} kareto_search_point;                /* 48 bytes */
/* out: host [cap] in evaluation order (rounds ascending, (d, t) ascending within a round);
 * *n_out = number evaluated; *truncated = 1 when a round would have exceeded cap or
 * max_rounds (that round is not evaluated, R40).  Errors: KARETO_E_INVALID (bad ranges /
 * steps / thresholds, t * 1000 >= 2^32 - 1 ms), plus those of kareto_eval_grid. */
kareto_status kareto_search(kareto_ctx *ctx, const kareto_trace *tr, const kareto_search_params *params,
                            const kareto_model *model, kareto_search_point *out, int64_t cap, int64_t *n_out,
                            int32_t *truncated);

/* ------------------------------------------------- row f2: group TTLs ---- */
/* Alg. 2 "ROI-Aware TTL Allocation" over the exact group curves of
 * P:750-752 for the loaded trace's K+1 groups (R23):
 *   H_g(t) = #{delta in Delta_g : delta <= t},  C_g(t) = |B_g| t + sum_{delta in Delta_g} min(t, delta),
 * Delta_g = the reuse intervals (ms) of the group's non-first accesses, |B_g| its unique blocks;
 * t in ms, C in block * ms.  All outputs are host arrays of K+1 entries (or n). */

/* Alg. 2 l.4-5: t_roi[g] = argmax over the candidate TTLs {max(delta, 1)} of H_g/C_g, exact,
 * ties -> smallest t, empty group -> 0 (R43); h_roi / c_roi (may be NULL) = H_g, C_g there. */
kareto_status kareto_ttl_roi(kareto_ctx *ctx, const kareto_trace *tr, uint32_t *t_roi, uint64_t *h_roi,
                             uint64_t *c_roi);
/* sum_g H_g(ttl[i][g]) and sum_g C_g(ttl[i][g]) for n TTL vectors ttl [n][K+1] (host, ms, finite;
 * KARETO_TTL_INF -> KARETO_E_INVALID naming the entry). */
kareto_status kareto_ttl_eval(kareto_ctx *ctx, const kareto_trace *tr, const uint32_t *ttl, int64_t n,
                              uint64_t *hits, uint64_t *cost);
/* Eq. 3 by Alg. 2: ROI TTLs, alpha = budget / sum C_g(t_roi) (R46), floor(sqrt(K))
 * deterministic perturbed starts from `seed` (R45), one start at the largest uniform TTL whose
 * cost fits the budget (R54), the exact discrete local solve from each
 * start (R44), the start with the most hits.  t_out = t*, hits_out / cost_out = its totals
 * (cost_out <= budget); t_roi_out / t_init_out may be NULL. */
kareto_status kareto_ttl_allocate(kareto_ctx *ctx, const kareto_trace *tr, uint64_t budget, uint64_t seed,
                                  uint32_t *t_out, uint64_t *hits_out, uint64_t *cost_out, uint32_t *t_roi_out,
                                  uint32_t *t_init_out);

/* ------------------------------------------------ row f3: queue model ---- */
/* Queue-coupled disk prefetch and per-request TTFT (PAPER.md Obs. 2/4; P99 TTFT
 * constraints), DESIGN R49-R53, for stack-eligible LRU configurations (TTL mode, or
 * CAPACITY with one TTL for every group): per request its prefix hits by tier (from the LRU
 * depths); FCFS over model->instances instances; a request's disk-resident prefix blocks count as
 * hits only if they stream in (at the medium's bandwidth) during its queue wait; TTFT = wait +
 * prefill + DRAM load.  out [n_cfg] host.  Errors: KARETO_E_INVALID (tuner / medium / TTL mode
 * with an infinite TTL / instances outside 1..4096), KARETO_E_UNSUPPORTED (non-LRU or per-group
 * TTLs on a finite disk: no stack path), _E_OOM. */
typedef struct {
  double ttft_mean_ms;          /* mean TTFT over requests                                  */
  double ttft_p99_ms;           /* nearest-rank P99 TTFT                                    */
  double makespan_s;            /* max(span, last instance free time)                       */
  double tokens_per_s;          /* (Ltok + O) / makespan                                    */
  uint64_t disk_hits_capacity;  /* disk-resident prefix blocks (capacity prediction)        */
  uint64_t disk_hits_realized;  /* of those, prefetched before service started              */
} kareto_queue_result;          /* 48 bytes */
kareto_status kareto_eval_queue(kareto_ctx *ctx, const kareto_trace *tr, const kareto_config *cfg, int64_t n_cfg,
                                const uint32_t *ttl_ms, int32_t n_tuner, const kareto_model *model,
                                kareto_queue_result *out);

/* ---------------------------------------- row f4: time-sharded trace passes ---- */
/* Collective over the ranks of ctx (world W <= 128, every rank passes the SAME desc): rank k
 * keeps the sorted requests [r_k, r_{k+1}) whose blocks cover positions ~[kN/W, (k+1)N/W) of
 * the touch order and runs the trace passes (K1 hash, K2 prev / delta / chain check / groups,
 * K3 LRU depth) on them only; with host inputs only that range of tokens is
 * copied.  Shard boundaries are crossed by an owner-partitioned exchange (three all-to-all-v:
 * first/last access records of every block, answers, the boundary LRU sets) and the groups /
 * counts by an allgather and an allreduce -- DESIGN.md "Time sharding".  Per access, prev
 * (global positions), delta and depth equal the whole-trace load's; U, U_g, reuse_g and groups
 * (of the shard's requests) too.  kareto_eval_grid on a time-sharded trace sums the K4
 * histograms over the ranks and returns the full grid on every rank; it accepts only
 * stack-path configurations (LRU with a uniform or TTL-mode disk TTL; others:
 * KARETO_E_UNSUPPORTED), and kareto_eval_queue / kareto_trace_analytics / kareto_ttl_* need a
 * whole trace (KARETO_E_UNSUPPORTED).  kareto_trace_export returns the shard's accesses.
 * Errors: as kareto_load_trace, plus KARETO_E_UNSUPPORTED (W > 128, requests of >= 2^24
 * blocks), _E_NCCL.  World 1: a whole trace computed by the sharded path. */
kareto_status kareto_load_trace_sharded(kareto_ctx *ctx, const kareto_trace_desc *desc, kareto_trace **out);
/* Host-only helpers (no device work) exposing the two partition rules of the time-sharded load:
 * req_bounds[k] (k = 0..world) = first sorted request whose first block position s[r] is >= k N / W
 * (N = s[R]), req_bounds[world] = R -- rank k keeps requests [req_bounds[k], req_bounds[k+1]);
 * s: host [R+1] block starts in sorted request order (kareto_trace_export KARETO_X_START).
 * kareto_hash_owner: the rank that owns a block hash in the exchange (top 32 bits of
 * fmix64(hash ^ 0x6A09E667F3BCC909) scaled to [0, world)); -1 if world < 1. */
kareto_status kareto_time_slices(const uint32_t *s, int64_t R, int32_t world, int64_t *req_bounds);
int32_t kareto_hash_owner(uint64_t block_hash, int32_t world);
/* The shard of a trace: sorted requests [*req_lo, *req_hi), positions [*pos_lo, *pos_hi)
 * (a whole trace: [0, R), [0, N)).  Any output may be NULL. */
kareto_status kareto_trace_shard(const kareto_trace *tr, int64_t *req_lo, int64_t *req_hi, int64_t *pos_lo,
                                 int64_t *pos_hi);

/* ------------------------------------------------ row f4: trace analytics ---- */
/* X6 reuse skew and X5 oracle-TTL footprint, DESIGN R47-R48:
 *   hits(b) = accesses of block b after its first; total_hits = sum; blocks sorted by hits
 *   descending; blocks_90 = fewest top blocks holding >= 90% of the hits (frac_90 = blocks_90 / U;
 *   no hits: blocks_90 = U, frac_90 = 1); lorenz[i] (i < n_pts) = share of the hits held by the
 *   top ceil(i U / (n_pts - 1)) blocks;
 *   after request r (arrival order): cumulative[r] = distinct blocks seen so far, active[r] =
 *   blocks seen so far whose next access is in a later request (the oracle TTL); peak_active =
 *   max_r active[r] at its first request peak_active_request.
 * lorenz [n_pts] (n_pts = 0 or >= 2), cumulative / active [R] are host arrays or NULL. */
typedef struct {
  int64_t unique_blocks, total_hits, blocks_90;
  double frac_90;
  int64_t peak_active, peak_active_request, final_cumulative;
} kareto_analytics;
kareto_status kareto_trace_analytics(kareto_ctx *ctx, const kareto_trace *tr, kareto_analytics *out, double *lorenz,
                                     int32_t n_pts, int64_t *cumulative, int64_t *active);

/* ------------------------------------------------------------ profiling ---- */
typedef struct {
  char name[24];      /* kernel / pass name                                         */
  double ms;          /* device time of the pass (CUDA events on the context stream),
                         summed over its launches                                  */
  int32_t launches;   /* number of timed launches of this pass                      */
  int32_t own;        /* 1: a kernel of this library; 0: a CUB primitive           */
} kareto_pass_time;
/* Enable (1) / disable (0) per-pass CUDA-event timing of subsequent calls. */
kareto_status kareto_set_profiling(kareto_ctx *ctx, int32_t on);
/* Per-pass device times accumulated (while profiling is on) by all calls since context
 * creation or the last reset; writes up to max entries and their number to *n; reset != 0
 * clears the accumulators after reading.  *own_launches (kareto_launch_counter) counts
 * launches of this library's own kernels (always on), reset the same way. */
kareto_status kareto_get_pass_times(kareto_ctx *ctx, kareto_pass_time *out, int32_t max, int32_t *n,
                                    int32_t reset);
kareto_status kareto_launch_counter(kareto_ctx *ctx, int64_t *own_launches, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* KARETO_H */

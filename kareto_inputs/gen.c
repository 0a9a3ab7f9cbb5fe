/*
 * kareto_inputs/gen.c -- seeded synthetic KV-block trace generator.
 *
 * This module is the ONLY code shared by the oracle (oracle/) and the CUDA path
 * (paper_2603_08739_b200/): both consume the arrays it fills.  It holds none of
 * the method's arithmetic -- no block hashing, no replay, no model -- only a
 * counter-based RNG, a few textbook distributions and the segment layout of the
 * synthetic sessions described in DESIGN.md "Input recipe" (after SURVEY 8.d.3).
 *
 * Trace shape follows the paper's workloads (PAPER.md 3.3, lines 368-374:
 * "Trace A: interactive chatbot workloads featuring multi-turn dialogues; Trace
 * B: programmatic API workloads; Trace C: agent-based workloads ... Each trace
 * spans 2 hours ... (16 tokens per block)"; "reuse intervals affected by
 * tool invocation durations").
 *
 * Output (file order = session order, NOT arrival order; consumers must sort):
 *   arrival_ms[R] int64, output_tokens[R] int32, offsets[R+1] int64, tokens[T] uint32.
 * A request's input is: [system prompt] + all earlier (user, output) segments of
 * its session + its own user segment.  Token ids of a segment are a pure
 * function of (seed, segment id, offset), so shared segments are identical and
 * all other content is unique.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KG_CHAT 0
#define KG_API 1
#define KG_AGENT 2

#define KG_VOCAB 151936u /* a realistic tokenizer vocabulary size */

/* ---- counter-based RNG (generator-private constants) ---------------------- */
static inline uint64_t kg_mix(uint64_t x) {
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ULL;
  x ^= x >> 32;
  x *= 0xd6e8feb86659fd93ULL;
  x ^= x >> 32;
  return x;
}
static inline uint64_t kg_rand(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return kg_mix(kg_mix(seed * 0xa0761d6478bd642fULL + stream) ^ (ctr * 0xe7037ed1a0b428dbULL + 0x8ebc6af09c88c6e3ULL));
}
typedef struct {
  uint64_t seed, stream, ctr;
} kg_rng;
static inline uint64_t kg_next(kg_rng *g) { return kg_rand(g->seed, g->stream, g->ctr++); }
static inline double kg_unif(kg_rng *g) { /* (0,1) */
  return ((double)(kg_next(g) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
static double kg_normal(kg_rng *g) {
  double u1 = kg_unif(g), u2 = kg_unif(g);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static int64_t kg_lognormal(kg_rng *g, double median, double sigma, int64_t lo, int64_t hi) {
  double v = median * exp(sigma * kg_normal(g));
  int64_t x = (int64_t)llround(v);
  if (x < lo) x = lo;
  if (x > hi) x = hi;
  return x;
}
static int64_t kg_unif_int(kg_rng *g, int64_t lo, int64_t hi) { /* inclusive */
  return lo + (int64_t)(kg_next(g) % (uint64_t)(hi - lo + 1));
}
static int64_t kg_geometric(kg_rng *g, double mean) { /* failures before success, E = mean */
  double p = 1.0 / (1.0 + mean);
  return (int64_t)floor(log(kg_unif(g)) / log(1.0 - p));
}
static int kg_zipf(kg_rng *g, const double *cdf, int n) {
  double u = kg_unif(g);
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (cdf[mid] >= u) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* ---- plan ------------------------------------------------------------------ */
typedef struct {
  int64_t session, turn;   /* session index, turn index in the session            */
  int64_t arrival_ms;
  int64_t input_len;       /* tokens                                               */
  int32_t output_len;
  int32_t sys_id;          /* -1: no system prompt                                 */
  int64_t tok_off;
} kg_req;

typedef struct {
  int kind;
  uint64_t seed;
  int n_pool;
  int64_t *pool_len;       /* system prompt pool lengths                          */
  int64_t n_req, cap_req;
  kg_req *req;
  /* per-session segment lengths (user_i, out_i), flattened */
  int64_t n_seg, cap_seg;
  int64_t *seg_len;        /* [2*turn] user, [2*turn+1] out                        */
  int64_t *sess_seg0;      /* first seg index of each session                     */
  int64_t n_sess, cap_sess;
  int64_t n_tokens, n_blocks;
} kg_plan;

static void *kg_grow(void *p, int64_t *cap, int64_t need, size_t elt) {
  if (need <= *cap) return p;
  int64_t c = *cap ? *cap : 1024;
  while (c < need) c *= 2;
  *cap = c;
  return realloc(p, (size_t)c * elt);
}

#define KG_CTX_CAP 131072
#define KG_SPAN_MS 7200000.0

int64_t kg_plan_requests(const kg_plan *p) { return p->n_req; }
int64_t kg_plan_tokens(const kg_plan *p) { return p->n_tokens; }
int64_t kg_plan_blocks(const kg_plan *p) { return p->n_blocks; }

void kg_plan_free(kg_plan *p) {
  if (!p) return;
  free(p->pool_len);
  free(p->req);
  free(p->seg_len);
  free(p->sess_seg0);
  free(p);
}

/*
 * kind: KG_CHAT (G-chat), KG_API (G-api), KG_AGENT (G-agent).
 * Generation stops once R_target requests exist (if R_target > 0) or once the
 * number of full 16-token blocks reaches N_target (if N_target > 0).
 */
kg_plan *kg_plan_create(int kind, int64_t R_target, int64_t N_target, uint64_t seed) {
  kg_plan *p = (kg_plan *)calloc(1, sizeof(kg_plan));
  p->kind = kind;
  p->seed = seed;
  /* system-prompt pool */
  double zipf_s;
  int64_t plo, phi;
  if (kind == KG_CHAT) { p->n_pool = 256; zipf_s = 1.1; plo = 256; phi = 1536; }
  else if (kind == KG_API) { p->n_pool = 32; zipf_s = 1.3; plo = 1024; phi = 8192; }
  else { p->n_pool = 16; zipf_s = 1.2; plo = 4096; phi = 16384; }
  p->pool_len = (int64_t *)malloc(sizeof(int64_t) * p->n_pool);
  double *cdf = (double *)malloc(sizeof(double) * p->n_pool);
  double z = 0;
  for (int i = 0; i < p->n_pool; i++) z += 1.0 / pow((double)(i + 1), zipf_s);
  double acc = 0;
  for (int i = 0; i < p->n_pool; i++) {
    acc += 1.0 / pow((double)(i + 1), zipf_s) / z;
    cdf[i] = acc;
    kg_rng g = {seed, 0x5157ULL, (uint64_t)i};
    p->pool_len[i] = kg_unif_int(&g, plo, phi);
  }
  cdf[p->n_pool - 1] = 1.0;

  int64_t sess = 0;
  for (;;) {
    if (R_target > 0 && p->n_req >= R_target) break;
    if (R_target <= 0 && p->n_blocks >= N_target) break;
    kg_rng g = {seed, 0x10000ULL + (uint64_t)sess, 0};
    int64_t start = (int64_t)floor(kg_unif(&g) * KG_SPAN_MS);
    int32_t sys_id = -1;
    int64_t turns;
    if (kind == KG_CHAT) {
      if (kg_unif(&g) < 0.7) sys_id = kg_zipf(&g, cdf, p->n_pool);
      turns = 1 + kg_geometric(&g, 2.0);
      if (turns > 64) turns = 64;
    } else if (kind == KG_API) {
      sys_id = kg_zipf(&g, cdf, p->n_pool);
      turns = 1;
    } else {
      sys_id = kg_zipf(&g, cdf, p->n_pool);
      turns = 1 + kg_geometric(&g, 15.0);
    }
    int64_t sys_len = sys_id >= 0 ? p->pool_len[sys_id] : 0;
    p->sess_seg0 = (int64_t *)kg_grow(p->sess_seg0, &p->cap_sess, sess + 1, sizeof(int64_t));
    p->sess_seg0[sess] = p->n_seg;
    int64_t ctx = sys_len, t_ms = start;
    for (int64_t t = 0; t < turns; t++) {
      int64_t u, o, gap;
      if (kind == KG_CHAT) {
        u = kg_lognormal(&g, 120.0, 1.0, 4, 8192);
        o = kg_lognormal(&g, 180.0, 0.8, 1, 4096);
        gap = kg_lognormal(&g, 30000.0, 1.0, 0, 3600000);
      } else if (kind == KG_API) {
        u = kg_lognormal(&g, 1500.0, 0.8, 16, 65536);
        o = kg_lognormal(&g, 150.0, 0.7, 1, 4096);
        gap = 0;
      } else {
        u = kg_lognormal(&g, 600.0, 1.0, 1, 32768);  /* task (t=0) / tool output */
        o = kg_lognormal(&g, 200.0, 0.8, 1, 4096);   /* model output */
        gap = kg_lognormal(&g, 4000.0, 1.2, 100, 600000);
      }
      if (ctx + u > KG_CTX_CAP) break;
      if (R_target > 0 && p->n_req >= R_target) break;
      p->seg_len = (int64_t *)kg_grow(p->seg_len, &p->cap_seg, p->n_seg + 2, sizeof(int64_t));
      p->seg_len[p->n_seg++] = u;
      p->seg_len[p->n_seg++] = o;
      p->req = (kg_req *)kg_grow(p->req, &p->cap_req, p->n_req + 1, sizeof(kg_req));
      kg_req *q = &p->req[p->n_req++];
      q->session = sess;
      q->turn = t;
      q->arrival_ms = t_ms;
      q->input_len = ctx + u;
      q->output_len = (int32_t)o;
      q->sys_id = sys_id;
      q->tok_off = p->n_tokens;
      p->n_tokens += q->input_len;
      p->n_blocks += q->input_len / 16;
      ctx += u + o;
      t_ms += gap;
    }
    sess++;
  }
  p->n_sess = sess;
  free(cdf);
  return p;
}

void kg_plan_fill_meta(const kg_plan *p, int64_t *arrival_ms, int32_t *output_tokens, int64_t *offsets) {
  for (int64_t r = 0; r < p->n_req; r++) {
    arrival_ms[r] = p->req[r].arrival_ms;
    output_tokens[r] = p->req[r].output_len;
    offsets[r] = p->req[r].tok_off;
  }
  offsets[p->n_req] = p->n_tokens;
}

static inline uint32_t kg_token(uint64_t seed, uint64_t seg_id, uint64_t off) {
  return (uint32_t)(kg_rand(seed ^ 0x70c3ULL, seg_id, off) % KG_VOCAB);
}

static void kg_fill_one(const kg_plan *p, int64_t r, uint32_t *out) {
  const kg_req *q = &p->req[r];
  int64_t pos = 0;
  if (q->sys_id >= 0) {
    int64_t L = p->pool_len[q->sys_id];
    uint64_t sid = 0x5000000000000000ULL | (uint64_t)q->sys_id;
    for (int64_t i = 0; i < L; i++) out[pos++] = kg_token(p->seed, sid, (uint64_t)i);
  }
  int64_t s0 = p->sess_seg0[q->session];
  for (int64_t t = 0; t <= q->turn; t++) {
    for (int which = 0; which < 2; which++) {
      if (t == q->turn && which == 1) break;
      int64_t L = p->seg_len[s0 + 2 * t + which];
      uint64_t sid = ((uint64_t)q->session << 16) | ((uint64_t)t << 1) | (uint64_t)which;
      for (int64_t i = 0; i < L; i++) out[pos++] = kg_token(p->seed, sid, (uint64_t)i);
    }
  }
}

typedef struct {
  const kg_plan *p;
  uint32_t *tokens;
  int64_t r0, r1;
} kg_job;
static void *kg_worker(void *arg) {
  kg_job *j = (kg_job *)arg;
  for (int64_t r = j->r0; r < j->r1; r++) kg_fill_one(j->p, r, j->tokens + j->p->req[r].tok_off);
  return NULL;
}

void kg_plan_fill_tokens(const kg_plan *p, uint32_t *tokens, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  kg_job jobs[256];
  int64_t per = (p->n_req + threads - 1) / threads;
  for (int t = 0; t < threads; t++) {
    jobs[t].p = p;
    jobs[t].tokens = tokens;
    jobs[t].r0 = t * per < p->n_req ? t * per : p->n_req;
    jobs[t].r1 = (t + 1) * per < p->n_req ? (t + 1) * per : p->n_req;
    pthread_create(&th[t], NULL, kg_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
}

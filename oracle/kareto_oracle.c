/*
 * oracle/kareto_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the Kareto
 * configuration-evaluation path (arXiv 2603.08739): trace -> chained block
 * hashes -> per-access reuse quantities -> per-configuration tier counts ->
 * fp64 objective vectors -> pruned Pareto frontier.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path in paper_2603_08739_b200/.
 *
 * Citations: P:<line> = /root/reference/PAPER.md, S:<line> = SPEC.md,
 * DESIGN.md R<n> = the numbered readings of the paper in DESIGN.md.
 *
 * Levels:
 *   O1 or_replay      literal per-configuration replay of the tiered store
 *                     (P:357 multi-tier placement / hit simulation; P:360
 *                     radix-tree prefix reuse; P:506 DRAM capacity + disk TTL;
 *                     P:745-752 TTL storage cost), R9-R24.
 *   O2 or_stack_*     sequential Fenwick LRU stack depths + the closed forms
 *                     of DESIGN.md "Stack path" (Mattson et al. 1970 stack
 *                     property); validated against O1 by the tests.
 *   model / prune / pareto: Eq. 1-2, Alg. 1 expansion test
 *                     (P:555-559), dominance, ParetoFilter.
 *
 * Parity status: every function here is pinned by tests in tests/test_oracle_*.py
 * (worked examples, textbook Belady strings, closed forms, brute force on tiny
 * traces, O1<->O2 agreement, SPEC arithmetic) except the fluid objective
 * model's *constants* (R25-R33: "parity with the paper's numbers
 * unpinned"; its structure is pinned by closed-form special cases).
 *
 * Build: gcc -O2 -ffp-contract=off -shared -fPIC (no FMA contraction, R33).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_E_INVALID = 1, OR_E_PARSE = 2, OR_E_CHAIN = 3, OR_E_OOM = 4, OR_E_OVERFLOW = 7 };
enum { OR_TOKENS = 0, OR_HASHES = 1 };
enum { OR_LRU = 0, OR_FIFO = 1, OR_LFU = 2 };
enum { T_NONE = 0, T_HBM = 1, T_DRAM = 2, T_DISK = 3 };

#define OR_INF_CAP UINT64_MAX
#define OR_INF_TTL UINT32_MAX
#define OR_NA UINT64_MAX

/* ----------------------------------------------------------------------------
 * Hash specification (R2; the paper only says "salted hash blocks
 * (16 tokens per block)", and "token-level KV-block hashes").
 * ------------------------------------------------------------------------- */
static uint64_t or_fmix64(uint64_t z) { /* splitmix64 output finaliser */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint32_t or_nh_key(int i) { return (uint32_t)or_fmix64((uint64_t)(i + 1)); }

/* content hash of one 16-token block: NH-style multilinear sum + finaliser */
static uint64_t or_content_hash(const uint32_t *t) {
  uint64_t acc = 0;
  for (int j = 0; j < 8; j++) {
    uint32_t a = t[2 * j] + or_nh_key(2 * j);
    uint32_t b = t[2 * j + 1] + or_nh_key(2 * j + 1);
    acc += (uint64_t)a * (uint64_t)b;
    acc += ((uint64_t)t[2 * j + 1] << 32) | (uint64_t)t[2 * j];
  }
  return or_fmix64(acc);
}
#define OR_CHAIN_R 0x9E3779B97F4A7C15ULL
#define OR_SALT_C 0x243F6A8885A308D3ULL

uint64_t or_fmix64_export(uint64_t z) { return or_fmix64(z); }
uint64_t or_content_hash_export(const uint32_t *t) { return or_content_hash(t); }

/* chained hashes of a token sequence: h_k = fmix(P_k), P_k = R*P_{k-1} + c_k */
void or_chain_hashes(const uint32_t *tokens, int64_t n_tokens, uint64_t salt, uint64_t *out) {
  int64_t n = n_tokens / 16;
  uint64_t P = or_fmix64(salt ^ OR_SALT_C);
  for (int64_t k = 0; k < n; k++) {
    P = P * OR_CHAIN_R + or_content_hash(tokens + 16 * k);
    out[k] = or_fmix64(P);
  }
}

/* ----------------------------------------------------------------------------
 * Trace (DESIGN.md "Oracle" O-1..O-6).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t R, N, U, span_ms;
  int K;
  uint64_t Ltok, O;
  int64_t *arr;      /* [R] arrival (sorted order) */
  int64_t *in_len;   /* [R] input tokens L_r */
  int64_t *out_len;  /* [R] */
  int64_t *nblk;     /* [R] full blocks n_r */
  int64_t *s;        /* [R+1] first touch position of request r */
  int64_t *order;    /* [R] sorted index -> file index */
  int32_t *grp;      /* [R] group of request */
  uint64_t *root;    /* [R] root hash (valid when nblk > 0) */
  /* touch order arrays [N] */
  uint64_t *hash;
  int32_t *req;
  int32_t *k;
  int64_t *prev;     /* -1 = first access */
  int64_t *delta;    /* -1 = infinity */
  int32_t *bid;      /* dense block id, first-occurrence order */
  int64_t *U_g, *reuse_g; /* [K+1] */
} or_trace;

typedef struct {
  int64_t n_requests;
  const int64_t *arrival_ms;
  const int32_t *output_tokens;
  int32_t mode;
  const int64_t *offsets;
  const uint32_t *tokens;
  const uint64_t *block_hash;
  const int64_t *input_tokens;
  uint64_t salt;
  int32_t top_k;
} or_trace_desc;

static const int64_t *g_sort_arr;
static int or_cmp_req(const void *a, const void *b) {
  int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
  if (g_sort_arr[i] != g_sort_arr[j]) return g_sort_arr[i] < g_sort_arr[j] ? -1 : 1;
  return i < j ? -1 : (i > j);
}

void or_trace_free(or_trace *t) {
  if (!t) return;
  free(t->arr); free(t->in_len); free(t->out_len); free(t->nblk); free(t->s); free(t->order);
  free(t->grp); free(t->root); free(t->hash); free(t->req); free(t->k); free(t->prev);
  free(t->delta); free(t->bid); free(t->U_g); free(t->reuse_g);
  free(t);
}

/* open-addressing map: 64-bit key -> int64 slot payload index */
typedef struct {
  uint64_t cap;
  uint64_t *key;
  int64_t *val;   /* -1 = empty */
} or_map;
static int or_map_init(or_map *m, int64_t n) {
  uint64_t c = 16;
  while (c < (uint64_t)(2 * n + 16)) c <<= 1;
  m->cap = c;
  m->key = (uint64_t *)malloc(sizeof(uint64_t) * c);
  m->val = (int64_t *)malloc(sizeof(int64_t) * c);
  if (!m->key || !m->val) return OR_E_OOM;
  for (uint64_t i = 0; i < c; i++) m->val[i] = -1;
  return OR_OK;
}
static int64_t *or_map_slot(or_map *m, uint64_t key, int *found) {
  uint64_t i = or_fmix64(key ^ 0x1234567ULL) & (m->cap - 1);
  for (;;) {
    if (m->val[i] < 0) { m->key[i] = key; *found = 0; return &m->val[i]; }
    if (m->key[i] == key) { *found = 1; return &m->val[i]; }
    i = (i + 1) & (m->cap - 1);
  }
}
static void or_map_free(or_map *m) { free(m->key); free(m->val); }

typedef struct { uint64_t hash; int64_t reuse; } or_root;
static int or_cmp_root(const void *a, const void *b) {
  const or_root *x = (const or_root *)a, *y = (const or_root *)b;
  if (x->reuse != y->reuse) return x->reuse > y->reuse ? -1 : 1; /* reuse desc */
  if (x->hash != y->hash) return x->hash < y->hash ? -1 : 1;     /* root hash asc */
  return 0;
}

int or_trace_build(const or_trace_desc *d, or_trace **out) {
  *out = NULL;
  int64_t R = d->n_requests;
  if (R < 1 || d->top_k < 0 || (d->mode != OR_TOKENS && d->mode != OR_HASHES)) return OR_E_INVALID;
  or_trace *t = (or_trace *)calloc(1, sizeof(or_trace));
  t->R = R;
  t->K = d->top_k;
  t->arr = (int64_t *)malloc(sizeof(int64_t) * R);
  t->in_len = (int64_t *)malloc(sizeof(int64_t) * R);
  t->out_len = (int64_t *)malloc(sizeof(int64_t) * R);
  t->nblk = (int64_t *)malloc(sizeof(int64_t) * R);
  t->s = (int64_t *)malloc(sizeof(int64_t) * (R + 1));
  t->order = (int64_t *)malloc(sizeof(int64_t) * R);
  t->grp = (int32_t *)malloc(sizeof(int32_t) * R);
  t->root = (uint64_t *)calloc(R, sizeof(uint64_t));
  /* O-1: stable sort by (arrival, file index) (R6) */
  for (int64_t i = 0; i < R; i++) {
    t->order[i] = i;
    if (d->output_tokens[i] < 0) { or_trace_free(t); return OR_E_INVALID; }
    if (d->offsets[i + 1] < d->offsets[i]) { or_trace_free(t); return OR_E_INVALID; }
  }
  g_sort_arr = d->arrival_ms;
  qsort(t->order, (size_t)R, sizeof(int64_t), or_cmp_req);
  /* O-2: blocks; full 16-token blocks only (R3) */
  t->s[0] = 0;
  for (int64_t r = 0; r < R; r++) {
    int64_t f = t->order[r];
    t->arr[r] = d->arrival_ms[f];
    t->out_len[r] = d->output_tokens[f];
    int64_t cnt = d->offsets[f + 1] - d->offsets[f];
    if (d->mode == OR_TOKENS) {
      t->in_len[r] = cnt;
      t->nblk[r] = cnt / 16;
    } else {
      t->nblk[r] = cnt;
      t->in_len[r] = d->input_tokens ? d->input_tokens[f] : 16 * cnt;
      if (t->in_len[r] < 16 * cnt) { or_trace_free(t); return OR_E_INVALID; }
    }
    t->Ltok += (uint64_t)t->in_len[r];
    t->O += (uint64_t)t->out_len[r];
    t->s[r + 1] = t->s[r] + t->nblk[r];
  }
  int64_t N = t->s[R];
  t->N = N;
  t->span_ms = t->arr[R - 1] - t->arr[0];
  if (t->span_ms < 1) t->span_ms = 1;
  int64_t Nalloc = N > 0 ? N : 1;
  t->hash = (uint64_t *)malloc(sizeof(uint64_t) * Nalloc);
  t->req = (int32_t *)malloc(sizeof(int32_t) * Nalloc);
  t->k = (int32_t *)malloc(sizeof(int32_t) * Nalloc);
  t->prev = (int64_t *)malloc(sizeof(int64_t) * Nalloc);
  t->delta = (int64_t *)malloc(sizeof(int64_t) * Nalloc);
  t->bid = (int32_t *)malloc(sizeof(int32_t) * Nalloc);
  /* O-3 hashing, O-5 touch order: request r, blocks k = n-1 .. 0 (leaf -> root) */
  uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (Nalloc));
  for (int64_t r = 0; r < R; r++) {
    int64_t f = t->order[r], n = t->nblk[r];
    if (n == 0) continue;
    if (d->mode == OR_TOKENS) or_chain_hashes(d->tokens + d->offsets[f], 16 * n, d->salt, tmp);
    else memcpy(tmp, d->block_hash + d->offsets[f], sizeof(uint64_t) * n);
    for (int64_t k = 0; k < n; k++) {
      int64_t j = t->s[r] + (n - 1 - k);
      t->hash[j] = tmp[k];
      t->req[j] = (int32_t)r;
      t->k[j] = (int32_t)k;
    }
    t->root[r] = tmp[0];
  }
  free(tmp);
  /* O-4 chain consistency + O-5 prev / delta + dense ids */
  or_map m;
  if (or_map_init(&m, N) != OR_OK) { or_trace_free(t); return OR_E_OOM; }
  int64_t *last = (int64_t *)malloc(sizeof(int64_t) * Nalloc);      /* by dense id */
  uint64_t *parent = (uint64_t *)malloc(sizeof(uint64_t) * Nalloc); /* by dense id */
  int32_t *kfirst = (int32_t *)malloc(sizeof(int32_t) * Nalloc);
  int64_t U = 0;
  int status = OR_OK;
  for (int64_t j = 0; j < N; j++) {
    int found;
    int64_t *slot = or_map_slot(&m, t->hash[j], &found);
    int kk = t->k[j];
    uint64_t par = kk > 0 ? t->hash[j + 1] : 0; /* parent = block k-1, touched right after */
    if (!found) {
      *slot = U;
      t->bid[j] = (int32_t)U;
      last[U] = j;
      parent[U] = par;
      kfirst[U] = kk;
      t->prev[j] = -1;
      t->delta[j] = -1;
      U++;
    } else {
      int64_t b = *slot;
      if (kfirst[b] != kk || parent[b] != par) { status = OR_E_CHAIN; break; }
      t->bid[j] = (int32_t)b;
      t->prev[j] = last[b];
      t->delta[j] = t->arr[t->req[j]] - t->arr[t->req[last[b]]];
      last[b] = j;
    }
  }
  or_map_free(&m);
  free(last); free(parent); free(kfirst);
  if (status != OR_OK) { or_trace_free(t); return status; }
  t->U = U;
  /* O-6 groups: top-K prefix subtrees by reuse, residual K (R23) */
  int K = t->K;
  t->U_g = (int64_t *)calloc(K + 1, sizeof(int64_t));
  t->reuse_g = (int64_t *)calloc(K + 1, sizeof(int64_t));
  int64_t *req_reuse = (int64_t *)calloc(R, sizeof(int64_t));
  int64_t *req_first = (int64_t *)calloc(R, sizeof(int64_t));
  for (int64_t j = 0; j < N; j++) {
    if (t->prev[j] >= 0) req_reuse[t->req[j]]++; else req_first[t->req[j]]++;
  }
  or_map rm;
  or_map_init(&rm, R);
  or_root *roots = (or_root *)malloc(sizeof(or_root) * R);
  int64_t nroots = 0;
  for (int64_t r = 0; r < R; r++) {
    if (t->nblk[r] == 0) continue;
    int found;
    int64_t *slot = or_map_slot(&rm, t->root[r], &found);
    if (!found) { *slot = nroots; roots[nroots].hash = t->root[r]; roots[nroots].reuse = 0; nroots++; }
    roots[*slot].reuse += req_reuse[r];
  }
  qsort(roots, (size_t)nroots, sizeof(or_root), or_cmp_root);
  or_map rank;
  or_map_init(&rank, nroots);
  for (int64_t i = 0; i < nroots; i++) {
    int found;
    int64_t *slot = or_map_slot(&rank, roots[i].hash, &found);
    *slot = i;
  }
  for (int64_t r = 0; r < R; r++) {
    int g = K;
    if (t->nblk[r] > 0) {
      int found;
      int64_t rk = *or_map_slot(&rank, t->root[r], &found);
      g = rk < K ? (int)rk : K;
    }
    t->grp[r] = g;
    t->U_g[g] += req_first[r];
    t->reuse_g[g] += req_reuse[r];
  }
  or_map_free(&rm);
  or_map_free(&rank);
  free(roots); free(req_reuse); free(req_first);
  *out = t;
  return OR_OK;
}

void or_trace_stats(const or_trace *t, int64_t *R, int64_t *N, int64_t *U, int64_t *span_ms,
                    uint64_t *Ltok, uint64_t *O, int64_t *U_g, int64_t *reuse_g) {
  *R = t->R; *N = t->N; *U = t->U; *span_ms = t->span_ms; *Ltok = t->Ltok; *O = t->O;
  for (int g = 0; g <= t->K; g++) { if (U_g) U_g[g] = t->U_g[g]; if (reuse_g) reuse_g[g] = t->reuse_g[g]; }
}

/* per-access export in touch order (for parity of the intermediate stages) */
void or_trace_export(const or_trace *t, uint64_t *hash, int64_t *prev, int64_t *delta, int32_t *req,
                     int32_t *k, int32_t *grp_req, int64_t *s) {
  for (int64_t j = 0; j < t->N; j++) {
    if (hash) hash[j] = t->hash[j];
    if (prev) prev[j] = t->prev[j];
    if (delta) delta[j] = t->delta[j];
    if (req) req[j] = t->req[j];
    if (k) k[j] = t->k[j];
  }
  for (int64_t r = 0; r < t->R; r++) { if (grp_req) grp_req[r] = t->grp[r]; }
  for (int64_t r = 0; r <= t->R; r++) { if (s) s[r] = t->s[r]; }
}

/* ----------------------------------------------------------------------------
 * Configurations and counts.
 * ------------------------------------------------------------------------- */
typedef struct {
  uint64_t cap[3];
  uint8_t policy, medium;
  uint16_t tuner;
  int32_t axis[3];
} or_config;

typedef struct {
  uint64_t hit[3], miss, evict[3], disk_writes, hit_pos_sum, bytetime_block_ms, resident_after_hole;
} or_counts;

/* ----------------------------------------------------------------------------
 * O1: literal replay (R9-R22).
 * ------------------------------------------------------------------------- */
typedef struct {
  int policy;
  int32_t *heap[4];     /* per tier (1..3) */
  int64_t n[4];
  int32_t *pos;         /* position of block in its tier heap */
  int32_t *eheap;       /* disk expiry heap */
  int64_t en;
  int32_t *epos;
  uint8_t *tier;
  int64_t *last_t, *last_seq, *ins_seq, *freq, *lease_t;
  uint8_t *seen;
  const uint32_t *tau;  /* per group TTL (ms) */
  const int32_t *gblk;  /* group of block */
} or_state;

/* policy key comparison: LRU last_seq, FIFO ins_seq, LFU (freq, last_seq) (R24) */
static int or_less(const or_state *S, int32_t a, int32_t b) {
  if (S->policy == OR_LRU) return S->last_seq[a] < S->last_seq[b];
  if (S->policy == OR_FIFO) return S->ins_seq[a] < S->ins_seq[b];
  if (S->freq[a] != S->freq[b]) return S->freq[a] < S->freq[b];
  return S->last_seq[a] < S->last_seq[b];
}
static void or_hswap(or_state *S, int t, int64_t i, int64_t j) {
  int32_t a = S->heap[t][i], b = S->heap[t][j];
  S->heap[t][i] = b; S->heap[t][j] = a;
  S->pos[b] = (int32_t)i; S->pos[a] = (int32_t)j;
}
static void or_hup(or_state *S, int t, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!or_less(S, S->heap[t][i], S->heap[t][p])) break;
    or_hswap(S, t, i, p);
    i = p;
  }
}
static void or_hdown(or_state *S, int t, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < S->n[t] && or_less(S, S->heap[t][l], S->heap[t][m])) m = l;
    if (r < S->n[t] && or_less(S, S->heap[t][r], S->heap[t][m])) m = r;
    if (m == i) break;
    or_hswap(S, t, i, m);
    i = m;
  }
}
static void or_hpush(or_state *S, int t, int32_t b) {
  int64_t i = S->n[t]++;
  S->heap[t][i] = b;
  S->pos[b] = (int32_t)i;
  or_hup(S, t, i);
}
static void or_hremove(or_state *S, int t, int32_t b) {
  int64_t i = S->pos[b], last = --S->n[t];
  if (i != last) {
    or_hswap(S, t, i, last);
    or_hup(S, t, i);
    or_hdown(S, t, i);
  }
  S->pos[b] = -1;
}
/* expiry heap (disk, CAPACITY mode, finite tau): key = last_t + tau[g] */
static int64_t or_exp(const or_state *S, int32_t b) { return S->last_t[b] + (int64_t)S->tau[S->gblk[b]]; }
static void or_eswap(or_state *S, int64_t i, int64_t j) {
  int32_t a = S->eheap[i], b = S->eheap[j];
  S->eheap[i] = b; S->eheap[j] = a; S->epos[b] = (int32_t)i; S->epos[a] = (int32_t)j;
}
static void or_eup(or_state *S, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (or_exp(S, S->eheap[i]) >= or_exp(S, S->eheap[p])) break;
    or_eswap(S, i, p);
    i = p;
  }
}
static void or_edown(or_state *S, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < S->en && or_exp(S, S->eheap[l]) < or_exp(S, S->eheap[m])) m = l;
    if (r < S->en && or_exp(S, S->eheap[r]) < or_exp(S, S->eheap[m])) m = r;
    if (m == i) break;
    or_eswap(S, i, m);
    i = m;
  }
}
static void or_epush(or_state *S, int32_t b) {
  int64_t i = S->en++;
  S->eheap[i] = b; S->epos[b] = (int32_t)i; or_eup(S, i);
}
static void or_eremove(or_state *S, int32_t b) {
  int64_t i = S->epos[b], last = --S->en;
  if (i != last) { or_eswap(S, i, last); or_eup(S, i); or_edown(S, i); }
  S->epos[b] = -1;
}

typedef struct {
  or_state *S;
  const uint64_t *cap;
  int ttl_mode, use_expiry;
  int64_t seq;
  or_counts *c;
} or_run;

static void or_enter(or_run *X, int t, int32_t b);
/* CASCADE(t): while |tier t| > cap[t] demote/drop the policy victim (R9, R16) */
static void or_cascade(or_run *X, int t) {
  or_state *S = X->S;
  while ((uint64_t)S->n[t] > X->cap[t - 1]) {
    int32_t v = S->heap[t][0];
    or_hremove(S, t, v);
    if (t == T_DISK && S->epos[v] >= 0) or_eremove(S, v);
    X->c->evict[t - 1] += 1;
    int next_exists = X->ttl_mode ? (t == T_HBM) : (t < T_DISK);
    if (next_exists) {
      X->seq += 1;
      S->ins_seq[v] = X->seq; /* last_seq kept */
      or_enter(X, t + 1, v);
      or_cascade(X, t + 1);
    } else {
      S->tier[v] = T_NONE; /* drop (frequency forgotten: re-entry restarts at 1) */
    }
  }
}
static void or_enter(or_run *X, int t, int32_t b) {
  or_state *S = X->S;
  S->tier[b] = (uint8_t)t;
  or_hpush(S, t, b);
  if (t == T_DISK && X->use_expiry && S->tau[S->gblk[b]] != OR_INF_TTL) or_epush(S, b);
}

/* One configuration, literal replay. tau_row[K+1] (ms, OR_INF_TTL = infinity).  lookup_tier
 * (may be NULL): [N] per access (touch order) the tier that served it in its request's hit
 * prefix (1 HBM, 2 DRAM, 3 disk or lease store), 0 outside the prefix (row f3, R51). */
int or_replay_lookup(const or_trace *tr, const or_config *cfg, const uint32_t *tau_row, or_counts *out,
                     uint8_t *lookup_tier) {
  memset(out, 0, sizeof(*out));
  if (cfg->policy > OR_LFU) return OR_E_INVALID;
  int ttl_mode = cfg->cap[2] == OR_INF_CAP;
  int any_finite = 0, all_finite = 1;
  for (int g = 0; g <= tr->K; g++) {
    if (tau_row[g] != OR_INF_TTL) any_finite = 1; else all_finite = 0;
  }
  if (ttl_mode && !all_finite) return OR_E_INVALID; /* DESIGN.md R22 */
  if (cfg->cap[0] == OR_INF_CAP || cfg->cap[1] == OR_INF_CAP) return OR_E_INVALID;
  int64_t U = tr->U > 0 ? tr->U : 1;
  or_state S;
  memset(&S, 0, sizeof(S));
  S.policy = cfg->policy;
  S.tau = tau_row;
  for (int t = 1; t <= 3; t++) {
    uint64_t c = t == 3 ? (ttl_mode ? 0 : cfg->cap[2]) : cfg->cap[t - 1];
    int64_t sz = (c + 2 < (uint64_t)U + 2) ? (int64_t)c + 2 : U + 2;
    S.heap[t] = (int32_t *)malloc(sizeof(int32_t) * sz);
  }
  S.pos = (int32_t *)malloc(sizeof(int32_t) * U);
  S.eheap = (int32_t *)malloc(sizeof(int32_t) * (U + 2));
  S.epos = (int32_t *)malloc(sizeof(int32_t) * U);
  S.tier = (uint8_t *)calloc(U, 1);
  S.seen = (uint8_t *)calloc(U, 1);
  S.last_t = (int64_t *)calloc(U, sizeof(int64_t));
  S.last_seq = (int64_t *)calloc(U, sizeof(int64_t));
  S.ins_seq = (int64_t *)calloc(U, sizeof(int64_t));
  S.freq = (int64_t *)calloc(U, sizeof(int64_t));
  S.lease_t = (int64_t *)calloc(U, sizeof(int64_t));
  int32_t *gblk = (int32_t *)malloc(sizeof(int32_t) * U);
  if (!S.tier || !S.last_t || !S.lease_t || !gblk) return OR_E_OOM;
  for (int64_t i = 0; i < U; i++) { S.pos[i] = -1; S.epos[i] = -1; }
  for (int64_t j = 0; j < tr->N; j++) gblk[tr->bid[j]] = tr->grp[tr->req[j]];
  S.gblk = gblk;
  or_run X = {&S, cfg->cap, ttl_mode, (!ttl_mode && any_finite), 0, out};
  int32_t *chain = (int32_t *)malloc(sizeof(int32_t) * (tr->N > 0 ? tr->N : 1));
  for (int64_t r = 0; r < tr->R; r++) {
    int64_t n = tr->nblk[r], a = tr->arr[r];
    if (n == 0) continue;
    int g = tr->grp[r];
    for (int64_t k = 0; k < n; k++) chain[k] = tr->bid[tr->s[r] + (n - 1 - k)];
    /* 1 PURGE (CAPACITY mode): every DISK block with a - last_t > tau[g] (R20) */
    if (X.use_expiry) {
      while (S.en > 0 && or_exp(&S, S.eheap[0]) < a) {
        int32_t v = S.eheap[0];
        or_eremove(&S, v);
        or_hremove(&S, T_DISK, v);
        S.tier[v] = T_NONE;
      }
    }
    /* 2 LOOKUP on the pre-request state (R10, R11) */
    int64_t h = 0;
    for (; h < n; h++) {
      int32_t b = chain[h];
      int present = S.tier[b] != T_NONE ||
                    (ttl_mode && S.seen[b] && (uint64_t)(a - S.lease_t[b]) <= (uint64_t)tau_row[g]);
      if (!present) break;
    }
    for (int64_t k = 0; k < n; k++) {
      int32_t b = chain[k];
      if (lookup_tier) lookup_tier[tr->s[r] + (n - 1 - k)] = 0;
      if (k < h) {
        int t = S.tier[b] != T_NONE ? S.tier[b] : T_DISK;
        out->hit[t - 1] += 1;
        out->hit_pos_sum += (uint64_t)k;
        if (lookup_tier) lookup_tier[tr->s[r] + (n - 1 - k)] = (uint8_t)t;
      } else {
        out->miss += 1;
        if (S.tier[b] != T_NONE) out->resident_after_hole += 1;
      }
      if (ttl_mode) {
        if (!S.seen[b] || (uint64_t)(a - S.lease_t[b]) > (uint64_t)tau_row[g]) out->disk_writes += 1;
      }
    }
    /* 3 UPDATE leaf -> root (R12) */
    for (int64_t k = n - 1; k >= 0; k--) {
      int32_t b = chain[k];
      X.seq += 1;
      if (S.tier[b] == T_HBM) {
        if (S.policy == OR_LRU) { S.last_seq[b] = X.seq; or_hdown(&S, T_HBM, S.pos[b]); }
        else if (S.policy == OR_LFU) { S.freq[b] += 1; S.last_seq[b] = X.seq; or_hdown(&S, T_HBM, S.pos[b]); }
      } else {
        if (S.tier[b] == T_DRAM || S.tier[b] == T_DISK) {
          int t = S.tier[b];
          or_hremove(&S, t, b);
          if (t == T_DISK && S.epos[b] >= 0) or_eremove(&S, b);
          S.freq[b] += 1; /* LFU count carried across tiers */
        } else {
          S.freq[b] = 1;
        }
        S.last_seq[b] = X.seq;
        S.ins_seq[b] = X.seq;
        or_enter(&X, T_HBM, b);
        or_cascade(&X, T_HBM);
      }
      /* TTL-mode lease integral: time covered since the previous access */
      if (ttl_mode && S.seen[b]) {
        int64_t dt = a - S.lease_t[b];
        out->bytetime_block_ms += (uint64_t)(dt < (int64_t)tau_row[g] ? dt : (int64_t)tau_row[g]);
      }
      S.last_t[b] = a;
      if (S.tier[b] == T_DISK && S.epos[b] >= 0) { /* demoted during its own cascade: refresh key */
        or_eup(&S, S.epos[b]);
        or_edown(&S, S.epos[b]);
      }
      S.lease_t[b] = a;
      S.seen[b] = 1;
    }
  }
  if (ttl_mode) {
    for (int64_t b = 0; b < tr->U; b++)
      if (S.seen[b]) out->bytetime_block_ms += (uint64_t)tau_row[gblk[b]]; /* last lease: a full tau (R21) */
    out->evict[2] = 0;
  } else {
    out->disk_writes = cfg->cap[2] > 0 ? out->evict[1] : 0;
    if (any_finite) out->evict[2] = OR_NA;
  }
  free(chain);
  for (int t = 1; t <= 3; t++) free(S.heap[t]);
  free(S.pos); free(S.eheap); free(S.epos); free(S.tier); free(S.seen); free(S.last_t);
  free(S.last_seq); free(S.ins_seq); free(S.freq); free(S.lease_t); free(gblk);
  return OR_OK;
}

int or_replay(const or_trace *tr, const or_config *cfg, const uint32_t *tau_row, or_counts *out) {
  return or_replay_lookup(tr, cfg, tau_row, out, NULL);
}

typedef struct {
  const or_trace *tr;
  const or_config *cfg;
  const uint32_t *ttl;
  int32_t n_tuner;
  or_counts *out;
  int32_t *st;
  int64_t i0, i1;
} or_job;
static void *or_replay_worker(void *arg) {
  or_job *J = (or_job *)arg;
  for (int64_t i = J->i0; i < J->i1; i++) {
    if (J->cfg[i].tuner >= J->n_tuner) { J->st[i] = OR_E_INVALID; continue; }
    J->st[i] = or_replay(J->tr, &J->cfg[i], J->ttl + (int64_t)J->cfg[i].tuner * (J->tr->K + 1), &J->out[i]);
  }
  return NULL;
}
/* configurations are independent: one thread per core over configs */
int or_replay_many(const or_trace *tr, const or_config *cfg, int64_t n, const uint32_t *ttl, int32_t n_tuner,
                   or_counts *out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 512) threads = 512;
  pthread_t th[512];
  or_job jobs[512];
  int32_t *st = (int32_t *)calloc(n > 0 ? n : 1, sizeof(int32_t));
  /* interleaved static split keeps long and short configs mixed */
  int64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; t++) {
    or_job J = {tr, cfg, ttl, n_tuner, out, st, t * per < n ? t * per : n, (t + 1) * per < n ? (t + 1) * per : n};
    jobs[t] = J;
    pthread_create(&th[t], NULL, or_replay_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  int s = OR_OK;
  for (int64_t i = 0; i < n; i++) if (st[i] != OR_OK) { s = st[i]; break; }
  free(st);
  return s;
}

/* ----------------------------------------------------------------------------
 * O2: LRU stack depths by a sequential Fenwick tree.
 * d = number of live positions in [prev, s_r) at request start; D = d + (n-1-k).
 * ------------------------------------------------------------------------- */
static void fw_add(int64_t *f, int64_t n, int64_t i, int64_t v) { for (i++; i <= n; i += i & -i) f[i] += v; }
static int64_t fw_sum(const int64_t *f, int64_t i) { int64_t s = 0; for (; i > 0; i -= i & -i) s += f[i]; return s; }

void or_stack_depth(const or_trace *tr, int64_t *d, int64_t *D) {
  int64_t N = tr->N;
  int64_t *f = (int64_t *)calloc(N + 1, sizeof(int64_t));
  for (int64_t r = 0; r < tr->R; r++) {
    int64_t s = tr->s[r], e = tr->s[r + 1];
    for (int64_t j = s; j < e; j++) {
      int64_t p = tr->prev[j];
      if (p < 0) { d[j] = -1; if (D) D[j] = -1; continue; }
      d[j] = fw_sum(f, s) - fw_sum(f, p); /* live positions in [p, s) */
      if (D) D[j] = d[j] + (j - s);
    }
    for (int64_t j = s; j < e; j++) {
      if (tr->prev[j] >= 0) fw_add(f, N, tr->prev[j], -1);
      fw_add(f, N, j, 1);
    }
  }
  free(f);
}

/* sorted key list with prefix sums, for #{key <= b} and sum of payload over them */
typedef struct {
  int64_t n;
  int64_t *key;
  uint64_t *pre; /* pre[i] = sum of payload of the first i keys */
} or_cdf;
typedef struct { int64_t key; uint64_t pay; } or_kp;
static int or_cmp_kp(const void *a, const void *b) {
  int64_t x = ((const or_kp *)a)->key, y = ((const or_kp *)b)->key;
  return x < y ? -1 : (x > y);
}
static void or_cdf_build(or_cdf *c, or_kp *v, int64_t n) {
  qsort(v, (size_t)n, sizeof(or_kp), or_cmp_kp);
  c->n = n;
  c->key = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  c->pre = (uint64_t *)malloc(sizeof(uint64_t) * (n + 1));
  c->pre[0] = 0;
  for (int64_t i = 0; i < n; i++) { c->key[i] = v[i].key; c->pre[i + 1] = c->pre[i] + v[i].pay; }
}
static int64_t or_cdf_count(const or_cdf *c, int64_t b) { /* #{key <= b} */
  int64_t lo = 0, hi = c->n;
  while (lo < hi) { int64_t m = (lo + hi) / 2; if (c->key[m] <= b) lo = m + 1; else hi = m; }
  return lo;
}
static void or_cdf_free(or_cdf *c) { free(c->key); free(c->pre); }

typedef struct {
  int64_t tau;  /* -1 = infinity */
  int g;        /* -1 = all groups */
  or_cdf cdf;   /* over reuse accesses with delta <= tau in group g: key d, payload k */
} or_filt;

typedef struct {
  const or_trace *tr;
  int64_t *d, *D;
  or_cdf Dc;          /* all accesses, key D (first accesses: +inf) */
  or_cdf *dg;         /* per group: key delta over reuse accesses, payload delta */
  or_filt *f;
  int nf, capf;
} or_stack;

static or_cdf *or_stack_filter(or_stack *st, int64_t tau, int g) {
  for (int i = 0; i < st->nf; i++) if (st->f[i].tau == tau && st->f[i].g == g) return &st->f[i].cdf;
  if (st->nf == st->capf) {
    st->capf = st->capf ? 2 * st->capf : 8;
    st->f = (or_filt *)realloc(st->f, sizeof(or_filt) * st->capf);
  }
  const or_trace *tr = st->tr;
  or_kp *v = (or_kp *)malloc(sizeof(or_kp) * (tr->N > 0 ? tr->N : 1));
  int64_t n = 0;
  for (int64_t j = 0; j < tr->N; j++) {
    if (tr->prev[j] < 0) continue;
    if (tau >= 0 && tr->delta[j] > tau) continue;
    if (g >= 0 && tr->grp[tr->req[j]] != g) continue;
    v[n].key = st->d[j];
    v[n].pay = (uint64_t)tr->k[j];
    n++;
  }
  or_filt *F = &st->f[st->nf++];
  F->tau = tau;
  F->g = g;
  or_cdf_build(&F->cdf, v, n);
  free(v);
  return &F->cdf;
}

or_stack *or_stack_create(const or_trace *tr) {
  or_stack *st = (or_stack *)calloc(1, sizeof(or_stack));
  st->tr = tr;
  int64_t N = tr->N > 0 ? tr->N : 1;
  st->d = (int64_t *)malloc(sizeof(int64_t) * N);
  st->D = (int64_t *)malloc(sizeof(int64_t) * N);
  or_stack_depth(tr, st->d, st->D);
  or_kp *v = (or_kp *)malloc(sizeof(or_kp) * N);
  for (int64_t j = 0; j < tr->N; j++) { v[j].key = st->D[j] < 0 ? INT64_MAX : st->D[j]; v[j].pay = 0; }
  or_cdf_build(&st->Dc, v, tr->N);
  st->dg = (or_cdf *)calloc(tr->K + 1, sizeof(or_cdf));
  for (int g = 0; g <= tr->K; g++) {
    int64_t n = 0;
    for (int64_t j = 0; j < tr->N; j++) {
      if (tr->prev[j] < 0 || tr->grp[tr->req[j]] != g) continue;
      v[n].key = tr->delta[j];
      v[n].pay = (uint64_t)tr->delta[j];
      n++;
    }
    or_cdf_build(&st->dg[g], v, n);
  }
  free(v);
  return st;
}
void or_stack_free(or_stack *st) {
  if (!st) return;
  free(st->d); free(st->D);
  or_cdf_free(&st->Dc);
  for (int g = 0; g <= st->tr->K; g++) or_cdf_free(&st->dg[g]);
  free(st->dg);
  for (int i = 0; i < st->nf; i++) or_cdf_free(&st->f[i].cdf);
  free(st->f);
  free(st);
}
void or_stack_export(const or_stack *st, int64_t *d, int64_t *D) {
  for (int64_t j = 0; j < st->tr->N; j++) { if (d) d[j] = st->d[j]; if (D) D[j] = st->D[j]; }
}

static uint64_t or_sat_add(uint64_t a, uint64_t b) { return a > UINT64_MAX - b ? UINT64_MAX : a + b; }

/* Stack-eligible iff LRU and (TTL mode, or CAPACITY with uniform tau) */
int or_stack_eligible(const or_trace *tr, const or_config *cfg, const uint32_t *tau_row) {
  if (cfg->policy != OR_LRU) return 0;
  if (cfg->cap[2] == OR_INF_CAP) return 1;
  for (int g = 1; g <= tr->K; g++) if (tau_row[g] != tau_row[0]) return 0;
  return 1;
}

int or_stack_counts(or_stack *st, const or_config *cfg, const uint32_t *tau_row, or_counts *c) {
  const or_trace *tr = st->tr;
  memset(c, 0, sizeof(*c));
  if (!or_stack_eligible(tr, cfg, tau_row)) return OR_E_INVALID;
  int ttl_mode = cfg->cap[2] == OR_INF_CAP;
  int64_t U = tr->U;
  uint64_t c1 = cfg->cap[0], c12 = or_sat_add(c1, cfg->cap[1]);
  int64_t b1 = c1 > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)c1;
  int64_t b12 = c12 > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)c12;
  or_cdf *all = or_stack_filter(st, -1, -1);
  int64_t n1 = or_cdf_count(all, b1), n12 = or_cdf_count(all, b12);
  c->hit[0] = (uint64_t)n1;
  c->hit[1] = (uint64_t)(n12 - n1);
  uint64_t hps = all->pre[n12];
  /* evictions: #{D > b} - min(b, U) */
  int64_t gt1 = tr->N - or_cdf_count(&st->Dc, b1), gt12 = tr->N - or_cdf_count(&st->Dc, b12);
  c->evict[0] = (uint64_t)(gt1 - (b1 < U ? b1 : U));
  c->evict[1] = (uint64_t)(gt12 - (b12 < U ? b12 : U));
  if (!ttl_mode) {
    uint64_t C = or_sat_add(c12, cfg->cap[2]);
    int64_t bC = C > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)C;
    int64_t tau = tau_row[0] == OR_INF_TTL ? -1 : (int64_t)tau_row[0];
    or_cdf *f = or_stack_filter(st, tau, -1);
    int64_t a = or_cdf_count(f, bC), b = or_cdf_count(f, b12);
    c->hit[2] = (uint64_t)(a - b);
    hps += f->pre[a] - f->pre[b];
    c->disk_writes = cfg->cap[2] > 0 ? c->evict[1] : 0;
    if (tau < 0) {
      int64_t gtC = tr->N - or_cdf_count(&st->Dc, bC);
      c->evict[2] = (uint64_t)(gtC - (bC < U ? bC : U));
    } else {
      c->evict[2] = OR_NA;
    }
  } else {
    uint64_t h3 = 0, w = 0, bt = 0;
    for (int g = 0; g <= tr->K; g++) {
      int64_t tau = (int64_t)tau_row[g];
      or_cdf *dg = &st->dg[g];
      int64_t ndel = or_cdf_count(dg, tau);            /* #{delta <= tau, g} */
      or_cdf *f = or_stack_filter(st, tau, g);
      int64_t nin = or_cdf_count(f, b12);              /* #{d <= c12, delta <= tau, g} */
      h3 += (uint64_t)(ndel - nin);
      hps += f->pre[f->n] - f->pre[nin];
      w += (uint64_t)tr->U_g[g] + (uint64_t)(dg->n - ndel);
      bt += (uint64_t)tr->U_g[g] * (uint64_t)tau + dg->pre[ndel] + (uint64_t)tau * (uint64_t)(dg->n - ndel);
    }
    c->hit[2] = h3;
    c->disk_writes = w;
    c->bytetime_block_ms = bt;
    c->evict[2] = 0;
  }
  c->hit_pos_sum = hps;
  c->miss = (uint64_t)tr->N - c->hit[0] - c->hit[1] - c->hit[2];
  return OR_OK;
}

/* ----------------------------------------------------------------------------
 * Objective model (Eq. 1-2; DESIGN.md "Objective model" R25-R33).
 * fp64, fixed evaluation order, no FMA contraction, no libm.
 * ------------------------------------------------------------------------- */
typedef struct { double bw_base, bw_slope, bw_max, price; } or_medium;
typedef struct { double breakpoint, rate, jump; } or_phi_seg;
typedef struct {
  int32_t instances, gpus_per_instance;
  uint64_t alpha_ps, beta_ps, dec_ps, block_bytes;
  double bw_dram, c_hw, p_hbm, p_dram, iops_per_block, ttl_prov_gb;
  int32_t n_media, n_phi;
  or_medium media[8];
  or_phi_seg phi[8];
} or_model;

static double or_max(double a, double b) { return a > b ? a : b; }
static double or_min(double a, double b) { return a < b ? a : b; }

double or_phi(const or_model *m, double u) { /* piecewise linear with jumps, right-continuous */
  double v = 0.0;
  for (int i = 0; i < m->n_phi; i++) {
    if (u >= m->phi[i].breakpoint) {
      double top = (i + 1 < m->n_phi) ? or_min(u, m->phi[i + 1].breakpoint) : u;
      v = (v + m->phi[i].jump) + m->phi[i].rate * (top - m->phi[i].breakpoint);
    }
  }
  return v;
}

int or_model_valid(const or_model *m) {
  if (m->instances < 1 || m->gpus_per_instance < 1 || m->block_bytes < 1 || !(m->bw_dram > 0)) return 0;
  if (m->n_media < 1 || m->n_media > 8 || m->n_phi < 0 || m->n_phi > 8) return 0;
  for (int i = 0; i < m->n_media; i++)
    if (!(m->media[i].bw_max > 0) || m->media[i].bw_base < 0 || m->media[i].bw_slope < 0 || m->media[i].price < 0) return 0;
  for (int i = 1; i < m->n_phi; i++) if (!(m->phi[i].breakpoint > m->phi[i - 1].breakpoint)) return 0;
  if (m->n_phi > 0 && m->phi[0].breakpoint != 0.0) return 0;
  if (m->c_hw < 0 || m->p_hbm < 0 || m->p_dram < 0 || m->iops_per_block < 0 || m->ttl_prov_gb < 0) return 0;
  return 1;
}

/* P0_ps = sum_r (alpha*L + beta*L*(L-1)/2): no-cache prefill cost in picoseconds */
int or_prefill_p0(const or_trace *tr, const or_model *m, uint64_t *P0) {
  unsigned __int128 acc = 0;
  for (int64_t r = 0; r < tr->R; r++) {
    unsigned __int128 L = (unsigned __int128)tr->in_len[r];
    acc += (unsigned __int128)m->alpha_ps * L;
    if (L > 0) acc += (unsigned __int128)m->beta_ps * ((L * (L - 1)) / 2);
  }
  if (acc > (unsigned __int128)UINT64_MAX) return OR_E_OVERFLOW;
  *P0 = (uint64_t)acc;
  return OR_OK;
}

static double or_gb(uint64_t c, uint64_t Bb) { return (double)(c * Bb) / 1e9; }

int or_objective(const or_trace *tr, const or_model *m, const or_config *cfg, const or_counts *c, double *f) {
  if (!or_model_valid(m) || cfg->medium >= m->n_media) return OR_E_INVALID;
  uint64_t P0;
  if (or_prefill_p0(tr, m, &P0) != OR_OK) return OR_E_OVERFLOW;
  int ttl_mode = cfg->cap[2] == OR_INF_CAP;
  uint64_t Bb = m->block_bytes;
  uint64_t Hc = c->hit[0] + c->hit[1] + c->hit[2];
  uint64_t S = 16 * m->alpha_ps * Hc + m->beta_ps * (256 * c->hit_pos_sum + 120 * Hc);
  double prefill_s = (double)(P0 - S) * 1e-12;
  double decode_s = (double)(m->dec_ps * tr->O) * 1e-12;
  const or_medium *md = &m->media[cfg->medium];
  double prov_gb = ttl_mode ? m->ttl_prov_gb : or_gb(cfg->cap[2], Bb);
  double bw_disk = or_min(md->bw_max, md->bw_base + md->bw_slope * prov_gb);
  double dram_s = (double)(c->hit[1] * Bb) / m->bw_dram;
  uint64_t io = c->hit[2] + c->disk_writes;
  double disk_s = io == 0 ? 0.0 : (double)(io * Bb) / bw_disk;
  double busy_s = (((prefill_s + decode_s) + dram_s) + disk_s) / (double)m->instances;
  double T_s = (double)tr->span_ms * 1e-3;
  double M_s = or_max(T_s, busy_s);
  f[0] = 1e3 * ((((prefill_s + dram_s) + disk_s) / (double)tr->R) + or_max(0.0, busy_s - T_s) / 2.0);
  f[1] = -((double)(tr->Ltok + tr->O) / M_s);
  double hours = M_s / 3600.0;
  double cost = (m->c_hw * (double)((int64_t)m->instances * m->gpus_per_instance)) * hours;
  cost = cost + (m->p_hbm * or_gb(cfg->cap[0], Bb)) * hours;
  cost = cost + (m->p_dram * or_gb(cfg->cap[1], Bb)) * hours;
  if (ttl_mode) cost = cost + (md->price * ((double)Bb / 1e9)) * ((double)c->bytetime_block_ms / 3.6e6);
  else cost = cost + (md->price * or_gb(cfg->cap[2], Bb)) * hours;
  double iops = ((double)io * m->iops_per_block) / M_s;
  cost = cost + (or_phi(m, iops) / 730.0) * hours;
  f[2] = cost;
  return OR_OK;
}

int or_objective_many(const or_trace *tr, const or_model *m, const or_config *cfg, const or_counts *c, int64_t n,
                      double *f) {
  for (int64_t i = 0; i < n; i++) {
    int s = or_objective(tr, m, &cfg[i], &c[i], f + 3 * i);
    if (s != OR_OK) return s;
  }
  return OR_OK;
}

/* the same, configurations split across host threads (each objective is independent) */
typedef struct { const or_trace *tr; const or_model *m; const or_config *cfg; const or_counts *c; int64_t i0, i1;
                 double *f; int status; } or_obj_job;
static void *or_obj_worker(void *a) {
  or_obj_job *j = (or_obj_job *)a;
  j->status = or_objective_many(j->tr, j->m, j->cfg + j->i0, j->c + j->i0, j->i1 - j->i0, j->f + 3 * j->i0);
  return NULL;
}
int or_objective_many_mt(const or_trace *tr, const or_model *m, const or_config *cfg, const or_counts *c, int64_t n,
                         double *f, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > n) threads = n > 0 ? (int)n : 1;
  pthread_t th[256];
  or_obj_job jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t] = (or_obj_job){tr, m, cfg, c, n * t / threads, n * (t + 1) / threads, f, OR_OK};
    pthread_create(&th[t], NULL, or_obj_worker, &jobs[t]);
  }
  int st = OR_OK;
  for (int t = 0; t < threads; t++) {
    pthread_join(th[t], NULL);
    if (jobs[t].status != OR_OK && st == OR_OK) st = jobs[t].status;
  }
  return st;
}

/* ----------------------------------------------------------------------------
 * Pruning (Alg. 1 expansion test P:555-559; R34) and
 * ParetoFilter (R35).  status: 2 pruned, 1 frontier, 0 dominated.
 * ------------------------------------------------------------------------- */
static const or_config *g_pc;
static int g_axis;
static int or_line_cmp(const void *A, const void *B) {
  int64_t i = *(const int64_t *)A, j = *(const int64_t *)B;
  const or_config *x = &g_pc[i], *y = &g_pc[j];
  int o1 = (g_axis + 1) % 3, o2 = (g_axis + 2) % 3;
  if (x->policy != y->policy) return x->policy < y->policy ? -1 : 1;
  if (x->medium != y->medium) return x->medium < y->medium ? -1 : 1;
  if (x->tuner != y->tuner) return x->tuner < y->tuner ? -1 : 1;
  if (x->axis[o1] != y->axis[o1]) return x->axis[o1] < y->axis[o1] ? -1 : 1;
  if (x->axis[o2] != y->axis[o2]) return x->axis[o2] < y->axis[o2] ? -1 : 1;
  if (x->axis[g_axis] != y->axis[g_axis]) return x->axis[g_axis] < y->axis[g_axis] ? -1 : 1;
  return i < j ? -1 : (i > j);
}
static int or_same_line(const or_config *x, const or_config *y, int a) {
  int o1 = (a + 1) % 3, o2 = (a + 2) % 3;
  return x->policy == y->policy && x->medium == y->medium && x->tuner == y->tuner && x->axis[o1] == y->axis[o1] &&
         x->axis[o2] == y->axis[o2];
}
static double or_fabs(double x) { return x < 0 ? -x : x; }

void or_prune(const double *f, const or_config *cfg, int64_t n, double tau_e, uint8_t *pruned) {
  memset(pruned, 0, (size_t)n);
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  for (int a = 0; a < 3; a++) {
    for (int64_t i = 0; i < n; i++) idx[i] = i;
    g_pc = cfg;
    g_axis = a;
    qsort(idx, (size_t)n, sizeof(int64_t), or_line_cmp);
    int64_t i = 0;
    while (i < n) {
      int64_t e = i + 1;
      while (e < n && or_same_line(&cfg[idx[i]], &cfg[idx[e]], a)) e++;
      int stopped = 0;
      for (int64_t j = i + 1; j < e; j++) {
        if (stopped) { pruned[idx[j]] = 1; continue; }
        double p = f[3 * idx[j - 1]], q = f[3 * idx[j]];
        double den = or_max(or_max(or_fabs(p), or_fabs(q)), 1e-9);
        double rel = (p - q) / den;
        if (rel <= tau_e) stopped = 1; /* j* = j: everything after it is pruned */
      }
      i = e;
    }
  }
  free(idx);
}

/* status of configurations [i0, i1): the O(n^2) definition, row by row */
static void or_pareto_rows(const double *f, int64_t n, const uint8_t *pruned, uint8_t *status, int64_t i0,
                           int64_t i1) {
  for (int64_t i = i0; i < i1; i++) {
    if (pruned && pruned[i]) { status[i] = 2; continue; }
    int dom = 0;
    for (int64_t j = 0; j < n && !dom; j++) {
      if (j == i || (pruned && pruned[j])) continue;
      const double *y = f + 3 * j, *x = f + 3 * i;
      if (y[0] <= x[0] && y[1] <= x[1] && y[2] <= x[2] && (y[0] < x[0] || y[1] < x[1] || y[2] < x[2])) dom = 1;
    }
    status[i] = dom ? 0 : 1;
  }
}

int64_t or_pareto(const double *f, int64_t n, const uint8_t *pruned, uint8_t *status) {
  or_pareto_rows(f, n, pruned, status, 0, n);
  int64_t nf = 0;
  for (int64_t i = 0; i < n; i++) nf += status[i] == 1;
  return nf;
}

/* the same, rows split across host threads (each row's status depends only on the inputs) */
typedef struct { const double *f; int64_t n; const uint8_t *pruned; uint8_t *status; int64_t i0, i1; } or_pareto_job;
static void *or_pareto_worker(void *a) {
  or_pareto_job *j = (or_pareto_job *)a;
  or_pareto_rows(j->f, j->n, j->pruned, j->status, j->i0, j->i1);
  return NULL;
}
int64_t or_pareto_mt(const double *f, int64_t n, const uint8_t *pruned, uint8_t *status, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (threads > n) threads = n > 0 ? (int)n : 1;
  pthread_t th[256];
  or_pareto_job jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t] = (or_pareto_job){f, n, pruned, status, n * t / threads, n * (t + 1) / threads};
    pthread_create(&th[t], NULL, or_pareto_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
  int64_t nf = 0;
  for (int64_t i = 0; i < n; i++) nf += status[i] == 1;
  return nf;
}

// ctx.cu -- context lifetime, device memory pool, NCCL bootstrap, pass timing, trace handles.
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

namespace kareto {

// NCCL is dlopen'ed (libnccl.so.2, normally already loaded by torch.distributed), so the
// library has no link-time NCCL dependency; a context created without an id never touches it.

static NcclApi *load_nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.h ? &api : nullptr;
  tried = true;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *n : names) {
    api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) return nullptr;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
  api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
  api.AllReduce = (decltype(api.AllReduce))dlsym(api.h, "ncclAllReduce");
  api.Send = (decltype(api.Send))dlsym(api.h, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(api.h, "ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
  if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy) {
    api.h = nullptr;
    return nullptr;
  }
  return &api;
}

// Every pass is also an NVTX range (header-only NVTX3: a no-op unless a tool such as Nsight
// Systems / ncu --nvtx injects itself), so profiles group kernels by the path's steps.
Pass::Pass(kareto_ctx *c, const char *name, int own, int launches) : ctx(c) {
  nvtxRangePushA(name);
  if (own) ctx->own_launches += launches;
  if (!ctx->profiling) return;
  for (size_t i = 0; i < ctx->passes.size(); i++)
    if (strncmp(ctx->passes[i].name, name, 23) == 0) { idx = (int)i; break; }
  if (idx < 0 && (int)ctx->passes.size() < kMaxPasses) {
    PassAcc p{};
    strncpy(p.name, name, 23);
    p.own = own;
    ctx->passes.push_back(p);
    idx = (int)ctx->passes.size() - 1;
  }
  if (idx < 0) return;
  ctx->passes[idx].launches += launches;
  auto take = [&]() {
    cudaEvent_t e;
    if (!ctx->event_pool.empty()) { e = ctx->event_pool.back(); ctx->event_pool.pop_back(); }
    else cudaEventCreate(&e);
    return e;
  };
  a = take();
  b = take();
  cudaEventRecord(a, ctx->stream);
}

Pass::~Pass() {
  nvtxRangePop();
  if (idx < 0 || !a) return;
  cudaEventRecord(b, ctx->stream);
  ctx->pending.push_back({idx, a, b});
}

void flush_pass_times(kareto_ctx *ctx) {
  for (auto &p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) ctx->passes[p.idx].ms += ms;
    ctx->event_pool.push_back(p.a);
    ctx->event_pool.push_back(p.b);
  }
  ctx->pending.clear();
  (void)cudaGetLastError();
}

kareto_status sync(kareto_ctx *ctx, const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return fail(ctx, KARETO_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  flush_pass_times(ctx);
  return KARETO_OK;
}

}  // namespace kareto

using namespace kareto;

extern "C" kareto_status kareto_nccl_unique_id(void *out128) {
  if (!out128) return KARETO_E_INVALID;
  NcclApi *api = load_nccl();
  if (!api) return KARETO_E_NCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return KARETO_E_NCCL;
  memcpy(out128, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return KARETO_OK;
}

static kareto_ctx *new_ctx(int device, void *cuda_stream, int rank, int world) {
  kareto_ctx *ctx = new kareto_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)cuda_stream;
  ctx->rank = rank;
  ctx->world = world;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  int l2 = 0;
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
  ctx->l2_bytes = (size_t)l2;
  // the device's stream-ordered pool with an unlimited release threshold keeps buffers cached
  // across calls; the large transient K6 / queue allocations are returned to the device after
  // each call (pool_trim), so other allocators in the process are not starved.  (A private pool
  // per context, destroyed with it, crashed in kareto_destroy when eight loopback ranks
  // tore down after full-size time-sharded loads.)
  if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&ctx->pool, device);
  if (e == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    e = cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    delete ctx;
    return nullptr;
  }
  return ctx;
}

namespace kareto {

kareto_status wave_budget(kareto_ctx *ctx, double frac, double *bytes) {
  size_t freeb = 0, totb = 0, rsv = 0, used = 0;
  KCUDA(ctx, cudaStreamSynchronize(ctx->stream));
  KCUDA(ctx, cudaMemGetInfo(&freeb, &totb));
  cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &rsv);
  cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemCurrent, &used);
  double b = frac * ((double)freeb + (double)(rsv > used ? rsv - used : 0));
  // loopback ranks share this GPU and size their waves at the same moment
  if (ctx->loop && ctx->world > 1) b /= (double)ctx->world;
  if (const char *o = getenv("KARETO_K6_BUDGET")) {
    const double v = atof(o);
    if (v > 0) b = v;
  }
  *bytes = b;
  return KARETO_OK;
}

void pool_trim(kareto_ctx *ctx) {
  if (cudaStreamSynchronize(ctx->stream) == cudaSuccess) cudaMemPoolTrimTo(ctx->pool, 0);
  (void)cudaGetLastError();
}

}  // namespace kareto

extern "C" kareto_status kareto_create(int device, void *cuda_stream, const void *nccl_unique_id, int rank, int world,
                                       kareto_ctx **out) {
  if (!out) return KARETO_E_INVALID;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_unique_id)) return KARETO_E_INVALID;
  kareto_ctx *ctx = new_ctx(device, cuda_stream, rank, world);
  if (!ctx) return KARETO_E_CUDA;
  // world > 1, or world == 1 with an id: a 1-rank communicator, so every collective of
  // eval_grid / the time-sharded load runs through NCCL on one GPU (the NCCL path's self-check)
  if (world > 1 || nccl_unique_id) {
    NcclApi *api = load_nccl();
    if (!api) { delete ctx; return KARETO_E_NCCL; }
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t comm;
    if (api->CommInitRank(&comm, world, id, rank) != ncclSuccess) {
      delete ctx;
      return KARETO_E_NCCL;
    }
    ctx->nccl = api;
    ctx->nccl_comm = comm;
  }
  *out = ctx;
  return KARETO_OK;
}

struct kareto_loopback;
extern "C" int32_t kareto_loopback_world(const kareto_loopback *g);

extern "C" kareto_status kareto_create_loopback(int device, void *cuda_stream, kareto_loopback *group, int rank,
                                                kareto_ctx **out) {
  if (!out || !group) return KARETO_E_INVALID;
  *out = nullptr;
  const int world = kareto_loopback_world(group);
  if (rank < 0 || rank >= world) return KARETO_E_INVALID;
  kareto_ctx *ctx = new_ctx(device, cuda_stream, rank, world);
  if (!ctx) return KARETO_E_CUDA;
  ctx->loop = group;
  *out = ctx;
  return KARETO_OK;
}

extern "C" void kareto_destroy(kareto_ctx *ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  flush_pass_times(ctx);
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->nccl_comm && ctx->nccl) ctx->nccl->CommDestroy((ncclComm_t)ctx->nccl_comm);
  if (ctx->h2d_scratch) {
    cudaFreeAsync(ctx->h2d_scratch, ctx->stream);
    ctx->h2d_scratch = nullptr;
  }
  if (ctx->k2_scratch) {
    cudaFreeAsync(ctx->k2_scratch, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
  }
  delete ctx;
}

extern "C" const char *kareto_last_error(const kareto_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

extern "C" kareto_status kareto_set_profiling(kareto_ctx *ctx, int32_t on) {
  if (!ctx) return KARETO_E_INVALID;
  ctx->profiling = on != 0;
  return KARETO_OK;
}

extern "C" kareto_status kareto_get_pass_times(kareto_ctx *ctx, kareto_pass_time *out, int32_t max, int32_t *n,
                                               int32_t reset) {
  if (!ctx || !n || (max > 0 && !out)) return KARETO_E_INVALID;
  cudaStreamSynchronize(ctx->stream);
  flush_pass_times(ctx);
  int k = 0;
  for (auto &p : ctx->passes) {
    if (k >= max) break;
    memset(&out[k], 0, sizeof(out[k]));
    strncpy(out[k].name, p.name, 23);
    out[k].ms = p.ms;
    out[k].launches = p.launches;
    out[k].own = p.own;
    k++;
  }
  *n = k;
  if (reset) ctx->passes.clear();
  return KARETO_OK;
}

extern "C" kareto_status kareto_launch_counter(kareto_ctx *ctx, int64_t *own_launches, int32_t reset) {
  if (!ctx) return KARETO_E_INVALID;
  if (own_launches) *own_launches = ctx->own_launches;
  if (reset) ctx->own_launches = 0;
  return KARETO_OK;
}

extern "C" void kareto_trace_free(kareto_trace *tr) {
  if (!tr) return;
  // uses only the trace's own copy of the stream: a trace may outlive its context
  void *ptrs[] = {tr->arr, tr->s, tr->grp, tr->hash, tr->req, tr->prev, tr->delta, tr->depth,
                  tr->blk, tr->gblk, tr->arr_rel, tr->inlen, tr->outlen, tr->runs};
  for (void *p : ptrs)
    if (p) cudaFreeAsync(p, tr->stream);
  cudaStreamSynchronize(tr->stream);
  (void)cudaGetLastError();
  delete tr;
}

extern "C" kareto_status kareto_trace_stats(const kareto_trace *tr, kareto_trace_info *info, int64_t *group_unique,
                                            int64_t *group_reuse) {
  if (!tr) return KARETO_E_INVALID;
  if (info) {
    info->n_requests = tr->R;
    info->n_accesses = tr->N;
    info->n_unique = tr->U;
    info->span_ms = tr->span_ms;
    info->input_tokens = tr->Ltok;
    info->output_tokens = tr->O;
    info->top_k = tr->K;
    info->max_blocks_per_request = tr->max_blocks;
  }
  for (int g = 0; g <= tr->K; g++) {
    if (group_unique) group_unique[g] = tr->U_g[g];
    if (group_reuse) group_reuse[g] = tr->reuse_g[g];
  }
  return KARETO_OK;
}

extern "C" kareto_status kareto_trace_export(kareto_ctx *ctx, const kareto_trace *tr, int32_t which, void *out) {
  if (!ctx || !tr || !out) return KARETO_E_INVALID;
  const void *src = nullptr;
  size_t bytes = 0;
  const size_t n = (size_t)(tr->pos_hi - tr->pos_lo);  // a time shard exports its own accesses
  switch (which) {
    case KARETO_X_HASH: src = tr->hash; bytes = 8 * n; break;
    case KARETO_X_PREV: src = tr->prev; bytes = 4 * n; break;
    case KARETO_X_DELTA: src = tr->delta; bytes = 4 * n; break;
    case KARETO_X_REQ: src = tr->req; bytes = 4 * n; break;
    case KARETO_X_DEPTH:
      if (kareto_status e = ensure_depth(ctx, const_cast<kareto_trace *>(tr))) return e;
      src = tr->depth; bytes = 4 * n; break;
    case KARETO_X_GROUP: src = tr->grp; bytes = 2 * (size_t)tr->R; break;
    case KARETO_X_START: src = tr->s; bytes = 4 * (size_t)(tr->R + 1); break;
    default: return fail(ctx, KARETO_E_INVALID, "unknown export %d", which);
  }
  if (bytes == 0) return KARETO_OK;
  KCUDA(ctx, cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return sync(ctx, "trace_export");
}

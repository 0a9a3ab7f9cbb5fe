// comm.cu -- collectives between the ranks of a context.
//
// Production: one process per GPU, NCCL over NVLink 5 / NVSwitch (allgather, allreduce and a
// grouped send/recv all-to-all-v, all enqueued on the context stream).
//
// Loopback: W contexts of ONE process on one device, driven by W host threads (one per rank),
// exchanging through each other's device buffers with host barriers.  It runs exactly the
// multi-rank code paths of the library (the sharded configuration evaluation and the
// time-sharded trace load) on a single GPU, so they can be parity-tested where only one GPU
// exists; the data movement is the only thing it replaces.
#include <condition_variable>
#include <mutex>

#include "internal.cuh"

struct kareto_loopback {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void *> ptr;             // per rank: published device buffer
  std::vector<std::vector<size_t>> off;      // per rank: published byte offsets (all-to-all-v)
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace kareto {

__global__ void k_sum_rows(const unsigned long long *__restrict__ rows, int W, size_t n,
                           unsigned long long *__restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long a = 0;
    for (int w = 0; w < W; w++) a += rows[(size_t)w * n + i];
    out[i] = a;
  }
}

static kareto_status nccl_check(kareto_ctx *ctx, ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return KARETO_OK;
  const char *m = ctx->nccl && ctx->nccl->GetErrorString ? ctx->nccl->GetErrorString(r) : "";
  return fail(ctx, KARETO_E_NCCL, "%s: %s", what, m);
}

kareto_status coll_allgather(kareto_ctx *ctx, const void *send, void *recv, size_t bytes) {
  cudaStream_t st = ctx->stream;
  if (ctx->world == 1 && !ctx->nccl) {
    if (bytes) KCUDA(ctx, cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
    return KARETO_OK;
  }
  if (ctx->nccl) {
    if (bytes == 0) return KARETO_OK;
    return nccl_check(ctx, ctx->nccl->AllGather(send, recv, bytes, ncclUint8, (ncclComm_t)ctx->nccl_comm, st),
                      "ncclAllGather");
  }
  kareto_loopback *g = ctx->loop;
  KCUDA(ctx, cudaStreamSynchronize(st));
  g->ptr[ctx->rank] = send;
  g->barrier();
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < ctx->world && bytes; r++) {
    cudaError_t e2 = cudaMemcpyAsync((char *)recv + (size_t)r * bytes, g->ptr[r], bytes, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = e2;
  }
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e3;
  g->barrier();  // peers may reuse their send buffers only after everyone has read them
  KCUDA(ctx, e);
  return KARETO_OK;
}

kareto_status coll_allgather_host(kareto_ctx *ctx, const void *send, void *recv, size_t bytes) {
  const int W = ctx->world;
  if (W == 1 && !ctx->nccl) {
    memcpy(recv, send, bytes);
    return KARETO_OK;
  }
  DBuf<uint8_t> ds, dr;
  KTRY(ds.alloc(ctx, bytes)); KTRY(dr.alloc(ctx, bytes * W));
  KCUDA(ctx, cudaMemcpyAsync(ds.p, send, bytes, cudaMemcpyHostToDevice, ctx->stream));
  KTRY(coll_allgather(ctx, ds.p, dr.p, bytes));
  KCUDA(ctx, cudaMemcpyAsync(recv, dr.p, bytes * W, cudaMemcpyDeviceToHost, ctx->stream));
  KCUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return KARETO_OK;
}

kareto_status coll_allreduce_u64(kareto_ctx *ctx, unsigned long long *buf, size_t n) {
  if ((ctx->world == 1 && !ctx->nccl) || n == 0) return KARETO_OK;
  if (ctx->nccl) {
    if (!ctx->nccl->AllReduce) return fail(ctx, KARETO_E_NCCL, "ncclAllReduce not available");
    return nccl_check(ctx, ctx->nccl->AllReduce(buf, buf, n, ncclUint64, ncclSum, (ncclComm_t)ctx->nccl_comm,
                                                ctx->stream), "ncclAllReduce");
  }
  DBuf<unsigned long long> rows;
  KTRY(rows.alloc(ctx, n * ctx->world));
  KTRY(coll_allgather(ctx, buf, rows.p, 8 * n));
  k_sum_rows<<<grid_for((int64_t)n, 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(rows.p, ctx->world, n, buf);
  ctx->own_launches++;
  return KARETO_OK;
}

kareto_status coll_alltoallv(kareto_ctx *ctx, const void *send, const std::vector<size_t> &send_off, void *recv,
                             const std::vector<size_t> &recv_off) {
  const int W = ctx->world, me = ctx->rank;
  cudaStream_t st = ctx->stream;
  if ((int)send_off.size() != W + 1 || (int)recv_off.size() != W + 1)
    return fail(ctx, KARETO_E_INVALID, "alltoallv: offsets need world + 1 entries");
  if (W == 1 && !ctx->nccl) {
    const size_t b = send_off[1] - send_off[0];
    if (b != recv_off[1] - recv_off[0]) return fail(ctx, KARETO_E_INVALID, "alltoallv: size mismatch");
    if (b) KCUDA(ctx, cudaMemcpyAsync(recv, (const char *)send + send_off[0], b, cudaMemcpyDeviceToDevice, st));
    return KARETO_OK;
  }
  if (ctx->nccl) {
    NcclApi *a = ctx->nccl;
    if (!a->Send || !a->Recv || !a->GroupStart || !a->GroupEnd)
      return fail(ctx, KARETO_E_NCCL, "ncclSend/ncclRecv not available");
    ncclComm_t comm = (ncclComm_t)ctx->nccl_comm;
    KTRY(nccl_check(ctx, a->GroupStart(), "ncclGroupStart"));
    for (int r = 0; r < W; r++) {
      const size_t sb = send_off[r + 1] - send_off[r], rb = recv_off[r + 1] - recv_off[r];
      if (sb) KTRY(nccl_check(ctx, a->Send((const char *)send + send_off[r], sb, ncclUint8, r, comm, st), "ncclSend"));
      if (rb) KTRY(nccl_check(ctx, a->Recv((char *)recv + recv_off[r], rb, ncclUint8, r, comm, st), "ncclRecv"));
    }
    return nccl_check(ctx, a->GroupEnd(), "ncclGroupEnd");
  }
  kareto_loopback *g = ctx->loop;
  KCUDA(ctx, cudaStreamSynchronize(st));
  g->ptr[me] = send;
  g->off[me] = send_off;
  g->barrier();
  bool mismatch = false;
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < W; r++) {
    const size_t b = g->off[r][me + 1] - g->off[r][me];
    if (b != recv_off[r + 1] - recv_off[r]) { mismatch = true; continue; }
    if (!b) continue;
    cudaError_t e2 = cudaMemcpyAsync((char *)recv + recv_off[r], (const char *)g->ptr[r] + g->off[r][me], b,
                                     cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = e2;
  }
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e3;
  g->barrier();
  KCUDA(ctx, e);
  if (mismatch) return fail(ctx, KARETO_E_INVALID, "alltoallv: receive sizes do not match the peers' sends");
  return KARETO_OK;
}

}  // namespace kareto

extern "C" kareto_status kareto_loopback_create(int32_t world, kareto_loopback **out) {
  if (!out || world < 1 || world > 1024) return KARETO_E_INVALID;
  kareto_loopback *g = new kareto_loopback();
  g->world = world;
  g->ptr.assign(world, nullptr);
  g->off.assign(world, std::vector<size_t>());
  *out = g;
  return KARETO_OK;
}

extern "C" void kareto_loopback_destroy(kareto_loopback *g) { delete g; }

extern "C" int32_t kareto_loopback_world(const kareto_loopback *g) { return g ? g->world : 0; }

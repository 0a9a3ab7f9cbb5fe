// sort_policy_bench.cu -- microbenchmark of the K2 sort shape (u32 key, u64 value, 1.06e8 pairs):
// CUB's default onesweep policy (8-bit digits, 4 passes) against custom tunings (11-bit digits,
// 3 passes).  Not part of the library; used to choose K2's sort policy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/sort_policy_bench.cu -o /tmp/sortbench
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#ifndef BEGIN_BIT
#define BEGIN_BIT 16  // K2 sorts the top 16 key bits only (2 passes); 0 = the full 32-bit sort
#endif

template <int BITS, int THREADS, int ITEMS>
struct Hub {
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = BITS;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, uint32_t, BITS>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, BITS>;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, uint64_t, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, BITS>;
    using ScanPolicy = cub::AgentScanPolicy<512, 23, uint32_t, cub::BLOCK_LOAD_WARP_TRANSPOSE, cub::LOAD_DEFAULT,
                                            cub::BLOCK_STORE_WARP_TRANSPOSE, cub::BLOCK_SCAN_RAKING_MEMOIZE>;
    using DownsweepPolicy = cub::AgentRadixSortDownsweepPolicy<512, 23, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                               cub::LOAD_DEFAULT, cub::RADIX_RANK_MATCH,
                                                               cub::BLOCK_SCAN_WARP_SCANS, 7>;
    using AltDownsweepPolicy = cub::AgentRadixSortDownsweepPolicy<256, 47, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                                  cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                                  cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using UpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 23, uint64_t, cub::LOAD_DEFAULT, 7>;
    using AltUpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 47, uint64_t, cub::LOAD_DEFAULT, 6>;
    using SingleTilePolicy = cub::AgentRadixSortDownsweepPolicy<256, 19, uint64_t, cub::BLOCK_LOAD_DIRECT,
                                                                cub::LOAD_LDG, cub::RADIX_RANK_MEMOIZE,
                                                                cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using SegmentedPolicy = cub::AgentRadixSortDownsweepPolicy<192, 39, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                               cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                               cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using AltSegmentedPolicy = cub::AgentRadixSortDownsweepPolicy<384, 11, uint64_t, cub::BLOCK_LOAD_TRANSPOSE,
                                                                  cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                                  cub::BLOCK_SCAN_WARP_SCANS, 5>;
  };
  using MaxPolicy = Policy1000;
};

__global__ void k_fill(uint32_t *k, uint64_t *v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    k[i] = (uint32_t)(z >> 32);
    v[i] = (z << 32) | (uint32_t)i;
  }
}

template <typename Hub_>
static float run(const char *name, uint32_t *k0, uint64_t *v0, uint32_t *k1, uint64_t *v1, uint32_t *kr, uint64_t *vr,
                 int64_t n, void *tmp, size_t tmp_bytes, int reps, bool check, const uint32_t *ref) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaMemcpy(k1, k0, 4 * n, cudaMemcpyDeviceToDevice);
    cudaMemcpy(v1, v0, 8 * n, cudaMemcpyDeviceToDevice);
    cub::DoubleBuffer<uint32_t> dk(k1, kr);
    cub::DoubleBuffer<uint64_t> dv(v1, vr);
    size_t tb = tmp_bytes;
    cudaEventRecord(a);
    cudaError_t e = cub::DispatchRadixSort<false, uint32_t, uint64_t, uint32_t, Hub_>::Dispatch(
        tmp, tb, dk, dv, (uint32_t)n, BEGIN_BIT, 32, true, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    if (e != cudaSuccess) { printf("%s: error %s\n", name, cudaGetErrorString(e)); return -1; }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
    if (check && r == 0) {
      std::vector<uint64_t> hv(n);
      cudaMemcpy(hv.data(), dv.Current(), 8 * n, cudaMemcpyDeviceToHost);
      std::vector<uint32_t> hk(n);
      cudaMemcpy(hk.data(), dk.Current(), 4 * n, cudaMemcpyDeviceToHost);
      std::vector<uint32_t> rk(n);
      cudaMemcpy(rk.data(), ref, 4 * n, cudaMemcpyDeviceToHost);
      bool ok = true;
      for (int64_t i = 1; i < n && ok; i++) {
        const uint32_t a = hk[i - 1] >> BEGIN_BIT, b = hk[i] >> BEGIN_BIT;
        ok = a < b || (a == b && (uint32_t)hv[i] > (uint32_t)hv[i - 1]);  // ordered, stable
      }
      printf("%s: %s\n", name, ok ? "sorted, stable" : "MISMATCH");
    }
  }
  printf("%-28s %8.3f ms  %6.1f GB/s (passes x 24 B)\n", name, best, 0.0);
  return best;
}

int main() {
  const int64_t n = 105899735;
  uint32_t *k0, *k1, *kr, *kref;
  uint64_t *v0, *v1, *vr, *vref;
  cudaMalloc(&k0, 4 * n); cudaMalloc(&k1, 4 * n); cudaMalloc(&kr, 4 * n); cudaMalloc(&kref, 4 * n);
  cudaMalloc(&v0, 8 * n); cudaMalloc(&v1, 8 * n); cudaMalloc(&vr, 8 * n); cudaMalloc(&vref, 8 * n);
  k_fill<<<148 * 8, 256>>>(k0, v0, n);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, kref, v0, vref, n, 0, 32);
  tmp_bytes = tmp_bytes * 4 + (256 << 20);
  void *tmp;
  cudaMalloc(&tmp, tmp_bytes);
  size_t tb = tmp_bytes;
  cub::DeviceRadixSort::SortPairs(tmp, tb, k0, kref, v0, vref, n, 0, 32);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    tb = tmp_bytes;
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, 32);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
  }
  printf("%-28s %8.3f ms (cub::DeviceRadixSort::SortPairs, not in place)\n", "default", best);
  run<Hub<8, 256, 32>>("bits8 t256 i32 (K2 now)", k0, v0, k1, v1, kr, vr, n, tmp, tmp_bytes, 5, true, kref);
  run<Hub<8, 384, 29>>("bits8 t384 i29", k0, v0, k1, v1, kr, vr, n, tmp, tmp_bytes, 5, false, kref);
  run<Hub<8, 128, 64>>("bits8 t128 i64", k0, v0, k1, v1, kr, vr, n, tmp, tmp_bytes, 5, false, kref);
  run<Hub<7, 256, 32>>("bits7 t256 i32", k0, v0, k1, v1, kr, vr, n, tmp, tmp_bytes, 5, false, kref);
  printf("done\n");
  return 0;
}

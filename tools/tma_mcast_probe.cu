// tma_mcast_probe.cu — does TMA multicast across a cluster raise the per-SM ingest above the
// ~44 GB/s/SM of tma_probe.cu? Each CTA of a cluster of C loads 1/C of every tile (128 rows x
// 64 cols bf16, 16 KB) with .multicast::cluster to all C CTAs, so each SM RECEIVES full tiles
// while L2 serves each byte once per cluster. Ring of NS stages; slot reuse is guarded by a
// cluster-wide "empty" barrier (count C) that every CTA arrives on remotely after it consumed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_mcast_probe tools/tma_mcast_probe.cu -lcuda
// Run:   tools/tma_mcast_probe <cluster C> <ctas> <stages>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void wait_par(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(bar),
               "r"(par)
               : "memory");
}

__global__ void __launch_bounds__(32, 1) probe(const __grid_constant__ CUtensorMap map, int C, int ns, int tiles_per_cluster,
                                                int col_blocks, int row_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  constexpr int kTile = 128 * 128;
  const uint32_t rank = cta_rank();
  const int cluster = blockIdx.x / C;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x != 0) return;
  const uint16_t mask = static_cast<uint16_t>((1u << C) - 1);
  const int rows_per = 128 / C;
  auto issue = [&](int i) {
    const int s = i % ns;
    const long long t = static_cast<long long>(cluster) * tiles_per_cluster + i;
    const int cb = static_cast<int>(t % col_blocks), rt = static_cast<int>((t / col_blocks) % row_tiles);
    // my full barrier expects the WHOLE tile (every CTA's slice lands here)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(kTile) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(smem + s * kTile + rank * rows_per * 128)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&full[s])), "r"(cb * 64), "r"(rt * 128 + static_cast<int>(rank) * rows_per),
        "h"(mask)
        : "memory");
  };
  for (int i = 0; i < ns && i < tiles_per_cluster; ++i) issue(i);
  for (int i = 0; i < tiles_per_cluster; ++i) {
    const int s = i % ns;
    wait_par(su32(&full[s]), (i / ns) & 1);
    // consumed: tell every CTA of the cluster that my copy of slot s is free
    for (int q = 0; q < C; ++q) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(&empty[s])), "r"(q));
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    }
    if (i + ns < tiles_per_cluster) {
      wait_par(su32(&empty[s]), (i / ns) & 1);  // all C copies of slot s consumed
      issue(i + ns);
    }
  }
  // drain: keep the CTA (and its smem) alive until peers stop writing into it
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int C = argc > 1 ? atoi(argv[1]) : 2;
  const int ctas = argc > 2 ? atoi(argv[2]) : 148;
  const int ns = argc > 3 ? atoi(argv[3]) : 8;
  const size_t bytes = 2ull << 30;
  const int K = 4096;
  const long long rows = bytes / (K * 2);
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)(128 / C)};
  cuuint32_t es[2] = {1, 1};
  reinterpret_cast<EncFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int col_blocks = K / 64;
  const int row_tiles = static_cast<int>(rows / 128);
  const long long total = static_cast<long long>(col_blocks) * row_tiles;
  const int clusters = ctas / C;
  const int tpc = static_cast<int>(total / clusters);
  const int smem = ns * 128 * 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int it = 0; it < 2; ++it) cudaLaunchKernelEx(&cfg, probe, map, C, ns, tpc, col_blocks, row_tiles);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, probe, map, C, ns, tpc, col_blocks, row_tiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double hbm = static_cast<double>(tpc) * clusters * 128 * 128;  // bytes read from memory
  const double delivered = hbm * C;                                    // bytes landing in smem
  printf("{\"cluster\": %d, \"ctas\": %d, \"stages\": %d, \"ms\": %.3f, \"read_GBs\": %.1f, \"delivered_GBs\": %.1f, "
         "\"delivered_GBs_per_sm\": %.1f, \"err\": \"%s\"}\n",
         C, clusters * C, ns, ms, hbm / ms / 1e6, delivered / ms / 1e6, delivered / ms / 1e6 / (clusters * C),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}

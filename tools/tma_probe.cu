// tma_probe.cu — calibration microbenchmark: how fast can one CTA per SM stream weight tiles
// into shared memory with TMA on this B200? (no compute; a ring of NS stages per CTA)
//   mode 0: 2-D tensor-map boxes of 64 cols x BOXR rows of a row-major [R][4096] bf16 matrix
//           (the swap-AB GEMM's weight-tile pattern), HBM-resident (buffer >> L2)
//   mode 1: 1-D bulk copies of the same byte count (contiguous)
//   mode 2: mode 0 over a 32 MB buffer (L2-resident re-reads, the activation-tile pattern)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu -lcuda
// Run:   /tmp/tma_probe <mode> <ctas> <stages> <box_rows> [issuers] [variant]
//   issuers: independent rings per CTA, one issuing warp each (is the cap per ring or per SM?)
//   variant: 0 = one issuing warp per ring, 1 = rings on lanes of one warp, 2 = as 0 with test_wait spins
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap map, const char* base, int mode,
                                                int ns, int box_rows, int tiles_per_cta, int col_blocks, int row_tiles,
                                                int variant) {
  extern __shared__ __align__(1024) uint8_t smem_all[];
  __shared__ uint64_t full_all[4][16];
  const int tile_bytes = box_rows * 128;
  // variant 0/2: one issuing thread per warp (ring = warp); variant 1: rings = lanes of warp 0
  // variant 3: one thread, one ring, each stage = `issuers` boxes on one mbarrier (the GEMM pattern)
  const int nb = variant == 3 ? blockDim.x / 32 : 1;
  const int rings = variant == 3 ? 1 : blockDim.x / 32;
  if (variant == 1 ? threadIdx.x >= rings : variant == 3 ? threadIdx.x != 0 : threadIdx.x % 32 != 0) return;
  const int ring = variant == 1 ? threadIdx.x : threadIdx.x / 32;
  uint64_t* full = full_all[ring];
  uint8_t* smem = smem_all + ring * ns * tile_bytes;
  for (int s = 0; s < ns; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue = [&](int i) {
    const int s = i % ns;
    const long long t = (static_cast<long long>(blockIdx.x) * rings + ring) * tiles_per_cta + i;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(tile_bytes * nb) : "memory");
    for (int b = 0; b < nb; ++b) {
    const long long tb = t * nb + b;
    uint8_t* dst = smem + (static_cast<long long>(s) * nb + b) * tile_bytes;
    if (mode == 1) {
      const char* src = base + tb % (static_cast<long long>(col_blocks) * row_tiles) * tile_bytes;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst)),
                   "l"(src), "r"(tile_bytes), "r"(su32(&full[s]))
                   : "memory");
    } else {
      const int cb = static_cast<int>(tb % col_blocks), rt = static_cast<int>((tb / col_blocks) % row_tiles);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              su32(dst)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&full[s])), "r"(cb * 64), "r"(rt * box_rows)
          : "memory");
    }
    }
  };
  for (int i = 0; i < ns && i < tiles_per_cta; ++i) issue(i);
  for (int i = 0; i < tiles_per_cta; ++i) {
    const int s = i % ns;
    const uint32_t par = (i / ns) & 1;
    if (variant == 2)
      asm volatile(
          "{\n\t.reg .pred p;\nV_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra V_%=;\n}" ::"r"(
              su32(&full[s])),
          "r"(par)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
              su32(&full[s])),
          "r"(par)
          : "memory");
    if (i + ns < tiles_per_cta) issue(i + ns);
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int ctas = argc > 2 ? atoi(argv[2]) : 148;
  const int ns = argc > 3 ? atoi(argv[3]) : 8;
  const int box_rows = argc > 4 ? atoi(argv[4]) : 128;
  const int rings = argc > 5 ? atoi(argv[5]) : 1;
  const int variant = argc > 6 ? atoi(argv[6]) : 0;
  const size_t bytes = mode == 2 ? (32ull << 20) : (2ull << 30);
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
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  reinterpret_cast<EncFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int tile_bytes = box_rows * 128;
  const int col_blocks = K / 64;
  const int row_tiles = static_cast<int>(rows / box_rows);
  const long long total_tiles = mode == 2 ? 8ll * col_blocks * row_tiles : static_cast<long long>(col_blocks) * row_tiles;
  const int tiles_per_cta = static_cast<int>(total_tiles / ctas / rings);  // per ring (variant 3: boxes per stage ride along)
  const int smem = rings * ns * tile_bytes;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int it = 0; it < 2; ++it) probe<<<ctas, 32 * rings, smem>>>(map, buf, mode, ns, box_rows, tiles_per_cta, col_blocks, row_tiles, variant);
  cudaEventRecord(a);
  probe<<<ctas, 32 * rings, smem>>>(map, buf, mode, ns, box_rows, tiles_per_cta, col_blocks, row_tiles, variant);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  // variant 3 moves `rings` boxes per stage from one ring: tiles_per_cta/rings stages of rings boxes
  const double moved = static_cast<double>(tiles_per_cta) * ctas * rings * tile_bytes;
  printf("{\"variant\": %d, \"mode\": %d, \"rings\": %d, \"ctas\": %d, \"stages\": %d, \"box_rows\": %d, \"inflight_KB_per_sm\": %d, \"ms\": %.3f, "
         "\"GBs\": %.1f, \"GBs_per_cta\": %.1f, \"err\": \"%s\"}\n",
         variant, mode, rings, ctas, ns, box_rows, rings * ns * tile_bytes / 1024, ms, moved / ms / 1e6, moved / ms / 1e6 / ctas,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// llama_kernels.cu — the small kernels of the Llama-style forwards that are not fused into
// the tcgen05 GEMM epilogues (tc_gemm.cu): deterministic weight init, embedding gather (+ the
// per-chunk sums of squares the next GEMM folds into its RMSNorm scale), and the final
// argmax_lowest reduction (toylm.cpp:9-16: ties -> lowest id) over per-tile partials.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "llama.cuh"

namespace faser {
namespace {

constexpr double kIrwinHallStd = 37837.226772;  // std of the sum of four U{0..65535}

__device__ __forceinline__ float gen_value(uint64_t base, int64_t i, float c) {
  const uint64_t r = lm_mix64(base + static_cast<uint64_t>(i) * 0x9e3779b97f4a7c15ull);
  const int s = static_cast<int>(r & 0xffff) + static_cast<int>((r >> 16) & 0xffff) +
                static_cast<int>((r >> 32) & 0xffff) + static_cast<int>(r >> 48);
  return __fmul_rn(static_cast<float>(s - 131070), c);
}

__host__ __device__ inline uint64_t tensor_base(uint64_t seed, uint32_t tag) {
  return lm_mix64(seed ^ lm_mix64(tag));
}

float scale_for(float std) { return static_cast<float>(static_cast<double>(std) / kIrwinHallStd); }

__global__ void init_matrix_kernel(__nv_bfloat16* w, int64_t n, uint64_t base, float c, int64_t off) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] = __float2bfloat16_rn(gen_value(base, off + i, c));
}

// Column slice [c0, c0 + kl) of a row-major [rows][k_full] tensor (row-parallel TP shards).
__global__ void init_cols_kernel(__nv_bfloat16* w, int64_t rows, int64_t k_full, int64_t c0, int64_t kl,
                                 uint64_t base, float c) {
  const int64_t n = rows * kl;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / kl, col = i % kl;
    w[i] = __float2bfloat16_rn(gen_value(base, r * k_full + c0 + col, c));
  }
}

// Interleaved gate/up: output row n of wgu = group n/128; within < 64 -> gate row, else up row.
__global__ void init_gate_up_kernel(__nv_bfloat16* w, int ffn, int d, uint64_t base_g,
                                    uint64_t base_u, float c, int64_t f0) {
  const int64_t n = 2ll * ffn * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / d, col = i % d;
    const int64_t grp = row / 128, within = row % 128;
    const bool up = within >= 64;
    const int64_t j = f0 + grp * 64 + (up ? within - 64 : within);  // global FFN row (TP shard offset f0)
    w[i] = __float2bfloat16_rn(gen_value(up ? base_u : base_g, j * d + col, c));
  }
}

__global__ void init_embedding_kernel(__nv_bfloat16* emb, const __nv_bfloat16* lm, int vocab, int d,
                                      uint32_t ga, uint32_t gb, float beta, uint64_t base_noise,
                                      float c, uint64_t base_hard, double hard_fraction) {
  const int64_t n = static_cast<int64_t>(vocab) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / d, col = i % d;
    int64_t g = (static_cast<uint64_t>(ga) * static_cast<uint64_t>(t) + gb) % static_cast<uint64_t>(vocab);
    // "hard" tokens: successor shifted by V/2 (exact: 53-bit integer -> double, power-of-two scale)
    const double u = static_cast<double>(lm_mix64(base_hard + static_cast<uint64_t>(t)) >> 11) * 0x1.0p-53;
    if (u < hard_fraction) g = (g + vocab / 2) % vocab;
    const float lv = __bfloat162float(lm[g * d + col]);
    emb[i] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(beta, lv), gen_value(base_noise, i, c)));
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 148 * 32 ? g : 148 * 32);
}

// One CTA of 128 threads per (row, 128-column chunk).
__global__ void __launch_bounds__(128) embed_kernel(const __nv_bfloat16* __restrict__ emb, RowsDev rows, int d,
                                                    int t_stride, float* __restrict__ x,
                                                    __nv_bfloat16* __restrict__ xb, float* __restrict__ ss) {
  __shared__ float red[4];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int r = blockIdx.x, c = blockIdx.y * 128 + threadIdx.x;
  if (r >= *rows.n_rows) return;
  const int tok = rows.row_tok[r];
  FASER_DCHECK(static_cast<unsigned>(tok) < kTokLimit, "FASER check: embed row %d token %d\n", r, tok);
  const __nv_bfloat16 e = emb[static_cast<int64_t>(tok) * d + c];
  const float v = __bfloat162float(e);
  x[static_cast<int64_t>(r) * d + c] = v;
  xb[static_cast<int64_t>(r) * d + c] = e;
  float q = v * v;
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  if (threadIdx.x == 0) ss[static_cast<int64_t>(blockIdx.y) * t_stride + r] = (red[0] + red[1]) + (red[2] + red[3]);
}

// One warp per row.
__global__ void argmax_reduce_kernel(int n_tiles, RowsDev rows, int t_stride, const float2* __restrict__ amax,
                                     int* __restrict__ out) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= *rows.n_rows) return;
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int m = lane; m < n_tiles; m += 32) {
    const float2 p = amax[static_cast<int64_t>(m) * t_stride + r];
    const int pi = __float_as_int(p.y);
    if (p.x > bv || (p.x == bv && pi < bi)) {
      bv = p.x;
      bi = pi;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) out[r] = bi;
}

}  // namespace

cudaError_t lm_init_matrix(__nv_bfloat16* w, int64_t n, uint64_t seed, uint32_t tag, float std,
                           cudaStream_t s, int64_t offset) {
  init_matrix_kernel<<<grid_for(n), 256, 0, s>>>(w, n, tensor_base(seed, tag), scale_for(std), offset);
  return cudaGetLastError();
}

cudaError_t lm_init_cols(__nv_bfloat16* w, int64_t rows, int64_t k_full, int64_t c0, int64_t kl, uint64_t seed,
                         uint32_t tag, float std, cudaStream_t s) {
  init_cols_kernel<<<grid_for(rows * kl), 256, 0, s>>>(w, rows, k_full, c0, kl, tensor_base(seed, tag),
                                                       scale_for(std));
  return cudaGetLastError();
}

cudaError_t lm_init_gate_up(__nv_bfloat16* wgu, int ffn, int d, uint64_t seed, uint32_t tag_layer,
                            float std, cudaStream_t s, int64_t f0) {
  init_gate_up_kernel<<<grid_for(2ll * ffn * d), 256, 0, s>>>(
      wgu, ffn, d, tensor_base(seed, kTagGate * 4096u + tag_layer),
      tensor_base(seed, kTagUp * 4096u + tag_layer), scale_for(std), f0);
  return cudaGetLastError();
}

cudaError_t lm_init_embedding(__nv_bfloat16* emb, const __nv_bfloat16* lm, const LlamaShape& m,
                              uint32_t ga, uint32_t gb, cudaStream_t s) {
  init_embedding_kernel<<<grid_for(static_cast<int64_t>(m.vocab) * m.d), 256, 0, s>>>(
      emb, lm, m.vocab, m.d, ga, gb, m.bigram_scale, tensor_base(m.seed, kTagEmbNoise * 4096u),
      scale_for(m.embed_noise), tensor_base(m.seed, kTagHard * 4096u), m.hard_fraction);
  return cudaGetLastError();
}

cudaError_t lm_embed(const LlamaShape& m, const __nv_bfloat16* emb, RowsDev rows, int rows_cap,
                     float* x, __nv_bfloat16* xb, float* ss, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  embed_kernel<<<dim3(rows_cap, m.d / 128), 128, 0, s>>>(emb, rows, m.d, rows_cap, x, xb, ss);
  return cudaGetLastError();
}

cudaError_t lm_argmax_reduce(int n_tiles, RowsDev rows, int rows_cap, const float2* amax, int* out,
                             cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  argmax_reduce_kernel<<<(rows_cap * 32 + 255) / 256, 256, 0, s>>>(n_tiles, rows, rows_cap, amax, out);
  return cudaGetLastError();
}

}  // namespace faser

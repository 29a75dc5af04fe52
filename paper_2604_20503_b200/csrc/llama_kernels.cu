// llama_kernels.cu — element-wise / row kernels of the Llama-style draft & verify forwards:
// deterministic weight init, embedding + RMSNorm, split-K reduction fused with RoPE + paged
// KV append, residual + RMSNorm, SwiGLU, logits reduction + argmax (lowest id on ties,
// argmax_lowest toylm.cpp:9-16). All are HBM/L2-bound row kernels; the projections
// themselves are the tcgen05 GEMM (tc_gemm.cu) and attention is llama_attn.cu.
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

__global__ void init_matrix_kernel(__nv_bfloat16* w, int64_t n, uint64_t base, float c) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w[i] = __float2bfloat16_rn(gen_value(base, i, c));
}

// Interleaved gate/up: output row n of wgu = group n/128; within < 64 -> gate row, else up row.
__global__ void init_gate_up_kernel(__nv_bfloat16* w, int ffn, int d, uint64_t base_g,
                                    uint64_t base_u, float c) {
  const int64_t n = 2ll * ffn * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / d, col = i % d;
    const int64_t grp = row / 128, within = row % 128;
    const bool up = within >= 64;
    const int64_t j = grp * 64 + (up ? within - 64 : within);
    w[i] = __float2bfloat16_rn(gen_value(up ? base_u : base_g, j * d + col, c));
  }
}

__global__ void init_embedding_kernel(__nv_bfloat16* emb, const __nv_bfloat16* lm, int vocab, int d,
                                      uint32_t ga, uint32_t gb, float beta, uint64_t base_noise,
                                      float c) {
  const int64_t n = static_cast<int64_t>(vocab) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / d, col = i % d;
    const int64_t g = (static_cast<uint64_t>(ga) * static_cast<uint64_t>(t) + gb) % static_cast<uint64_t>(vocab);
    const float lv = __bfloat162float(lm[g * d + col]);
    emb[i] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(beta, lv), gen_value(base_noise, i, c)));
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 148 * 32 ? g : 148 * 32);
}

// ------------------------------------------------------------------ block reductions
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

constexpr int kRowThreads = 256;

__global__ void __launch_bounds__(kRowThreads) embed_norm_kernel(
    const __nv_bfloat16* __restrict__ emb, RowsDev rows, int d, float eps, float* __restrict__ x,
    __nv_bfloat16* __restrict__ xn) {
  __shared__ float red[kRowThreads / 32];
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  const int tok = rows.row_tok[r];
  const __nv_bfloat16* e = emb + static_cast<int64_t>(tok) * d;
  float* xr = x + static_cast<int64_t>(r) * d;
  float ss = 0.f;
  for (int c = threadIdx.x; c < d; c += kRowThreads) {
    const float v = __bfloat162float(e[c]);
    xr[c] = v;
    ss += v * v;
  }
  ss = block_sum<kRowThreads>(ss, red);
  const float inv = rsqrtf(ss / d + eps);
  __nv_bfloat16* o = xn + static_cast<int64_t>(r) * d;
  for (int c = threadIdx.x; c < d; c += kRowThreads) o[c] = __float2bfloat16_rn(xr[c] * inv);
}

__global__ void __launch_bounds__(kRowThreads) residual_norm_kernel(
    const float* __restrict__ ws, int splits, int64_t split_stride, RowsDev rows, int d, float eps,
    float* __restrict__ x, __nv_bfloat16* __restrict__ xn) {
  __shared__ float red[kRowThreads / 32];
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  float* xr = x + static_cast<int64_t>(r) * d;
  const float* p = ws + static_cast<int64_t>(r) * d;
  float ss = 0.f;
  for (int c = threadIdx.x; c < d; c += kRowThreads) {
    float a = 0.f;
    for (int z = 0; z < splits; ++z) a += p[z * split_stride + c];
    const float v = xr[c] + a;
    xr[c] = v;
    ss += v * v;
  }
  ss = block_sum<kRowThreads>(ss, red);
  const float inv = rsqrtf(ss / d + eps);
  if (xn) {
    __nv_bfloat16* o = xn + static_cast<int64_t>(r) * d;
    for (int c = threadIdx.x; c < d; c += kRowThreads) o[c] = __float2bfloat16_rn(xr[c] * inv);
  }
}

// One CTA per row. Threads walk (head, i) pairs with i < hd/2 (rotate-half RoPE).
__global__ void __launch_bounds__(kRowThreads) qkv_rope_append_kernel(
    const float* __restrict__ ws, int splits, int64_t split_stride, RowsDev rows, int n_q, int n_kv,
    int hd, const float2* __restrict__ rope, KvDev kv, int layer, __nv_bfloat16* __restrict__ qbuf) {
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  const int half = hd / 2;
  const int nout = (n_q + 2 * n_kv) * hd;
  const int pos = rows.row_pos[r];
  const int slot = rows.req_slot[rows.row_req[r]];
  const int page = kv.ptab[static_cast<int64_t>(slot) * kv.max_pages + pos / kPage];
  const int off = pos % kPage;
  const float* p = ws + static_cast<int64_t>(r) * nout;
  const float2* rp = rope + static_cast<int64_t>(pos) * half;
  __nv_bfloat16* kvl = kv.pool + layer * kv.layer_stride;
  const int heads = n_q + 2 * n_kv;
  for (int e = threadIdx.x; e < heads * half; e += kRowThreads) {
    const int h = e / half, i = e % half;
    const int c0 = h * hd + i, c1 = c0 + half;
    float a = 0.f, b = 0.f;
    for (int z = 0; z < splits; ++z) {
      a += p[z * split_stride + c0];
      b += p[z * split_stride + c1];
    }
    if (h < n_q + n_kv) {  // rotate q and k
      const float2 cs = rp[i];
      const float ra = a * cs.x - b * cs.y;
      const float rb = b * cs.x + a * cs.y;
      a = ra;
      b = rb;
    }
    if (h < n_q) {
      __nv_bfloat16* q = qbuf + static_cast<int64_t>(r) * n_q * hd + h * hd;
      q[i] = __float2bfloat16_rn(a);
      q[i + half] = __float2bfloat16_rn(b);
    } else {
      const bool is_v = h >= n_q + n_kv;
      const int kvh = is_v ? h - n_q - n_kv : h - n_q;
      __nv_bfloat16* dst = kvl + ((static_cast<int64_t>(page) * n_kv + kvh) * 2 + (is_v ? 1 : 0)) * kPage * hd +
                           off * hd;
      dst[i] = __float2bfloat16_rn(a);
      dst[i + half] = __float2bfloat16_rn(b);
    }
  }
}

__global__ void __launch_bounds__(kRowThreads) swiglu_kernel(const float* __restrict__ ws, int splits,
                                                             int64_t split_stride, RowsDev rows,
                                                             int ffn, __nv_bfloat16* __restrict__ h) {
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  const float* p = ws + static_cast<int64_t>(r) * 2 * ffn;
  for (int j = threadIdx.x; j < ffn; j += kRowThreads) {
    const int grp = j / 64, w = j % 64;
    const int cg = grp * 128 + w, cu = cg + 64;
    float g = 0.f, u = 0.f;
    for (int z = 0; z < splits; ++z) {
      g += p[z * split_stride + cg];
      u += p[z * split_stride + cu];
    }
    const float s = g / (1.f + __expf(-g));
    h[static_cast<int64_t>(r) * ffn + j] = __float2bfloat16_rn(s * u);
  }
}

// Sums the split partials into split 0 (the logits [rows][vocab]) and takes argmax_lowest.
__global__ void __launch_bounds__(kRowThreads) logits_argmax_kernel(float* __restrict__ ws, int splits,
                                                                    int64_t split_stride, RowsDev rows,
                                                                    int vocab, int* __restrict__ out) {
  __shared__ float sv[kRowThreads / 32];
  __shared__ int si[kRowThreads / 32];
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  float* p = ws + static_cast<int64_t>(r) * vocab;
  float bv = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int v = threadIdx.x; v < vocab; v += kRowThreads) {
    float a = p[v];
    for (int z = 1; z < splits; ++z) a += p[z * split_stride + v];
    if (splits > 1) p[v] = a;
    if (a > bv) {  // increasing v per thread: strict '>' keeps the lowest id
      bv = a;
      bi = v;
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
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = bv;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bv = sv[0];
    bi = si[0];
    for (int i = 1; i < kRowThreads / 32; ++i)
      if (sv[i] > bv || (sv[i] == bv && si[i] < bi)) {
        bv = sv[i];
        bi = si[i];
      }
    out[r] = bi;
  }
}

}  // namespace

cudaError_t lm_init_matrix(__nv_bfloat16* w, int64_t n, uint64_t seed, uint32_t tag, float std,
                           cudaStream_t s) {
  init_matrix_kernel<<<grid_for(n), 256, 0, s>>>(w, n, tensor_base(seed, tag), scale_for(std));
  return cudaGetLastError();
}

cudaError_t lm_init_gate_up(__nv_bfloat16* wgu, int ffn, int d, uint64_t seed, uint32_t tag_layer,
                            float std, cudaStream_t s) {
  init_gate_up_kernel<<<grid_for(2ll * ffn * d), 256, 0, s>>>(
      wgu, ffn, d, tensor_base(seed, kTagGate * 4096u + tag_layer),
      tensor_base(seed, kTagUp * 4096u + tag_layer), scale_for(std));
  return cudaGetLastError();
}

cudaError_t lm_init_embedding(__nv_bfloat16* emb, const __nv_bfloat16* lm, const LlamaShape& m,
                              uint32_t ga, uint32_t gb, cudaStream_t s) {
  init_embedding_kernel<<<grid_for(static_cast<int64_t>(m.vocab) * m.d), 256, 0, s>>>(
      emb, lm, m.vocab, m.d, ga, gb, m.bigram_scale, tensor_base(m.seed, kTagEmbNoise * 4096u),
      scale_for(m.embed_noise));
  return cudaGetLastError();
}

cudaError_t lm_embed_norm(const LlamaShape& m, const __nv_bfloat16* emb, RowsDev rows, int rows_cap,
                          float* x, __nv_bfloat16* xn, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  embed_norm_kernel<<<rows_cap, kRowThreads, 0, s>>>(emb, rows, m.d, m.eps, x, xn);
  return cudaGetLastError();
}

cudaError_t lm_qkv_rope_append(const LlamaShape& m, const float* ws, int splits, int t_stride,
                               RowsDev rows, int rows_cap, const float2* rope, KvDev kv, int layer,
                               __nv_bfloat16* qbuf, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  qkv_rope_append_kernel<<<rows_cap, kRowThreads, 0, s>>>(
      ws, splits, static_cast<int64_t>(t_stride) * m.qkv_out(), rows, m.n_q, m.n_kv, m.hd, rope, kv,
      layer, qbuf);
  return cudaGetLastError();
}

cudaError_t lm_residual_norm(const LlamaShape& m, const float* ws, int splits, int t_stride,
                             RowsDev rows, int rows_cap, float* x, __nv_bfloat16* xn, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  residual_norm_kernel<<<rows_cap, kRowThreads, 0, s>>>(ws, splits, static_cast<int64_t>(t_stride) * m.d,
                                                        rows, m.d, m.eps, x, xn);
  return cudaGetLastError();
}

cudaError_t lm_swiglu(const LlamaShape& m, const float* ws, int splits, int t_stride, RowsDev rows,
                      int rows_cap, __nv_bfloat16* h, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  swiglu_kernel<<<rows_cap, kRowThreads, 0, s>>>(ws, splits, static_cast<int64_t>(t_stride) * 2 * m.ffn,
                                                 rows, m.ffn, h);
  return cudaGetLastError();
}

cudaError_t lm_logits_argmax(int vocab, float* ws, int splits, int t_stride, RowsDev rows,
                             int rows_cap, int* argmax_out, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  logits_argmax_kernel<<<rows_cap, kRowThreads, 0, s>>>(ws, splits, static_cast<int64_t>(t_stride) * vocab,
                                                        rows, vocab, argmax_out);
  return cudaGetLastError();
}

}  // namespace faser

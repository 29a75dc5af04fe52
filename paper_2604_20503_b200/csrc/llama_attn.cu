// llama_attn.cu — K3: varlen causal attention over the paged KV cache.
//
// Each request contributes n_i query rows at consecutive positions pos0_i .. pos0_i+n_i-1
// (1 row per draft step, k_i rows per verify, len-1 rows at prefill). GQA packing: the G
// query heads sharing a KV head are packed with the rows into the MMA M dimension
// (m = row*G + g), so a verify of k_i+... rows x 8 heads is one or a few 16-row tiles and the
// KV page is read once per (request, kv head) tile. QK^T and PV run on mma.sync bf16
// (m16n8k16, fp32 accumulate); K/V pages (64 tokens x head_dim, contiguous) are staged into
// XOR-swizzled shared memory with cp.async, double-buffered.
// Two work splits:
//   KEYS mode (few query rows, decode/verify): the 4 warps share one 16-row M tile and split
//            each 64-key page 4 ways; partial softmax states are merged through smem.
//   ROWS mode (>= 64 packed rows, long verify / prefill): each warp owns a 16-row M tile and
//            walks all keys of the page.
// Long contexts with few CTAs are split over KV (flash-decoding); a combine kernel merges.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "llama.cuh"

namespace faser {
namespace {

constexpr float kNegBig = -1e30f;

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled smem tile [64 keys][HD] bf16: 16-byte chunk c of row r lives at chunk c ^ (r & 7).
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
  return row * (HD * 2) + ((chunk ^ (row & 7)) << 4);
}

template <int HD, bool ROWS>
__global__ void __launch_bounds__(128) attn_kernel(RowsDev rows, KvDev kv, int layer, int n_q, int n_kv,
                                                   const __nv_bfloat16* __restrict__ qbuf,
                                                   __nv_bfloat16* __restrict__ obuf, float* __restrict__ part_o,
                                                   float2* __restrict__ part_ml, int n_split, int rows_cap,
                                                   float scale_log2) {
  constexpr int kChunks = HD / 8;          // 16-byte chunks per K/V row
  constexpr int kTileBytes = 64 * HD * 2;  // one K (or V) page
  constexpr int kKS = HD / 16;             // k-steps over head_dim
  constexpr int kDT = HD / 8;              // 8-wide dim tiles of O
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sK[2] = {smem, smem + 2 * kTileBytes};
  uint8_t* sV[2] = {smem + kTileBytes, smem + 3 * kTileBytes};

  const int req = blockIdx.x, kvh = blockIdx.y;
  const int nr = rows.req_n[req];
  const int G = n_q / n_kv;
  const int M = nr * G;
  const int blk = blockIdx.z / n_split, sp = blockIdx.z % n_split;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta_m0 = ROWS ? blk * 64 : blk * 16;
  if (cta_m0 >= M) return;
  const int cta_m1 = min(M, cta_m0 + (ROWS ? 64 : 16));
  const int first = rows.req_first[req], pos0 = rows.req_pos0[req];
  const int slot = rows.req_slot[req];
  const int key_end = pos0 + (cta_m1 - 1) / G + 1;
  const int tiles = (key_end + 63) / 64;
  const int tps = (tiles + n_split - 1) / n_split;
  const int t0 = sp * tps, t1 = min(tiles, t0 + tps);

  // ---- Q fragments of this warp's 16-row tile
  const int mt0 = ROWS ? cta_m0 + warp * 16 : cta_m0;
  const int mlo = mt0 + (lane >> 2), mhi = mlo + 8;
  uint32_t qa[kKS][4];
  {
    const int rlo = mlo / G, glo = mlo % G, rhi = mhi / G, ghi = mhi % G;
    const bool vlo = mlo < M, vhi = mhi < M;
    const __nv_bfloat16* qlo = qbuf + (static_cast<int64_t>(first + (vlo ? rlo : 0)) * n_q + kvh * G + glo) * HD;
    const __nv_bfloat16* qhi = qbuf + (static_cast<int64_t>(first + (vhi ? rhi : 0)) * n_q + kvh * G + ghi) * HD;
#pragma unroll
    for (int kk = 0; kk < kKS; ++kk) {
      const int c = kk * 16 + (lane & 3) * 2;
      qa[kk][0] = vlo ? *reinterpret_cast<const uint32_t*>(qlo + c) : 0u;
      qa[kk][1] = vhi ? *reinterpret_cast<const uint32_t*>(qhi + c) : 0u;
      qa[kk][2] = vlo ? *reinterpret_cast<const uint32_t*>(qlo + c + 8) : 0u;
      qa[kk][3] = vhi ? *reinterpret_cast<const uint32_t*>(qhi + c + 8) : 0u;
    }
  }
  const int lim_lo = pos0 + mlo / G, lim_hi = pos0 + mhi / G;  // last visible key per row

  float o[kDT][4];
#pragma unroll
  for (int i = 0; i < kDT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_lo = kNegBig, m_hi = kNegBig, l_lo = 0.f, l_hi = 0.f;

  const __nv_bfloat16* kvl = kv.pool + layer * kv.layer_stride;
  auto load_tile = [&](int t, int buf) {
    const int page = kv.ptab[static_cast<int64_t>(slot) * kv.max_pages + t];
    const uint8_t* gk = reinterpret_cast<const uint8_t*>(kvl + (static_cast<int64_t>(page) * n_kv + kvh) * 2 * 64 * HD);
    const uint8_t* gv = gk + kTileBytes;
#pragma unroll
    for (int i = threadIdx.x; i < 64 * kChunks; i += 128) {
      const int r = i / kChunks, c = i % kChunks;
      cp_async16(sK[buf] + swz<HD>(r, c), gk + i * 16);
      cp_async16(sV[buf] + swz<HD>(r, c), gv + i * 16);
    }
    cp_async_commit();
  };

  if (t0 < t1) load_tile(t0, 0);
  for (int t = t0; t < t1; ++t) {
    const int buf = (t - t0) & 1;
    if (t + 1 < t1) {
      load_tile(t + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint8_t* k_s = sK[buf];
    const uint8_t* v_s = sV[buf];
#pragma unroll
    for (int cc = 0; cc < (ROWS ? 4 : 1); ++cc) {
      const int c = ROWS ? cc : warp;  // 16-key chunk of the page
      const int kbase = t * 64 + c * 16;
      // S = Q K^T over 16 keys (two n-tiles of 8)
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < kKS; ++kk) {
        uint32_t b[4];
        const int mi = lane >> 3;
        const int key = c * 16 + 8 * (mi >> 1) + (lane & 7);
        ldsm_x4(b, k_s + swz<HD>(key, kk * 2 + (mi & 1)));
        mma16816(s[0], qa[kk], b[0], b[1]);
        mma16816(s[1], qa[kk], b[2], b[3]);
      }
      // scale, causal mask, online softmax
      float mx_lo = kNegBig, mx_hi = kNegBig;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = kbase + nt * 8 + (lane & 3) * 2 + e;
          s[nt][e] = key <= lim_lo ? s[nt][e] * scale_log2 : -INFINITY;
          s[nt][2 + e] = key <= lim_hi ? s[nt][2 + e] * scale_log2 : -INFINITY;
          mx_lo = fmaxf(mx_lo, s[nt][e]);
          mx_hi = fmaxf(mx_hi, s[nt][2 + e]);
        }
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, off));
        mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, off));
      }
      const float nm_lo = fmaxf(m_lo, mx_lo), nm_hi = fmaxf(m_hi, mx_hi);
      const float al_lo = exp2f(m_lo - nm_lo), al_hi = exp2f(m_hi - nm_hi);
      m_lo = nm_lo;
      m_hi = nm_hi;
      float p[2][4];
      float sl = 0.f, sh = 0.f;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        p[nt][0] = exp2f(s[nt][0] - nm_lo);
        p[nt][1] = exp2f(s[nt][1] - nm_lo);
        p[nt][2] = exp2f(s[nt][2] - nm_hi);
        p[nt][3] = exp2f(s[nt][3] - nm_hi);
        sl += p[nt][0] + p[nt][1];
        sh += p[nt][2] + p[nt][3];
      }
      l_lo = l_lo * al_lo + sl;
      l_hi = l_hi * al_hi + sh;
#pragma unroll
      for (int i = 0; i < kDT; ++i) {
        o[i][0] *= al_lo;
        o[i][1] *= al_lo;
        o[i][2] *= al_hi;
        o[i][3] *= al_hi;
      }
      uint32_t pa[4];
      pa[0] = pack_bf16(p[0][0], p[0][1]);
      pa[1] = pack_bf16(p[0][2], p[0][3]);
      pa[2] = pack_bf16(p[1][0], p[1][1]);
      pa[3] = pack_bf16(p[1][2], p[1][3]);
      // O += P V over the 16 keys
#pragma unroll
      for (int dt = 0; dt < kDT; dt += 2) {
        uint32_t b[4];
        const int mi = lane >> 3;
        const int key = c * 16 + 8 * (mi & 1) + (lane & 7);
        ldsm_x4_t(b, v_s + swz<HD>(key, dt + (mi >> 1)));
        mma16816(o[dt], pa, b[0], b[1]);
        mma16816(o[dt + 1], pa, b[2], b[3]);
      }
    }
    __syncthreads();
  }
  // quad-reduce the row sums
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, off);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, off);
  }

  if (!ROWS) {
    // merge the 4 warps' partial states (same 16 rows, disjoint keys) through smem
    float* so = reinterpret_cast<float*>(smem);             // [4][16][HD]
    float* sm = so + 4 * 16 * HD;                           // [4][16] m
    float* sl = sm + 64;                                    // [4][16] l
    const int rl = lane >> 2, rh = rl + 8;
#pragma unroll
    for (int dt = 0; dt < kDT; ++dt) {
      const int col = dt * 8 + (lane & 3) * 2;
      so[(warp * 16 + rl) * HD + col] = o[dt][0];
      so[(warp * 16 + rl) * HD + col + 1] = o[dt][1];
      so[(warp * 16 + rh) * HD + col] = o[dt][2];
      so[(warp * 16 + rh) * HD + col + 1] = o[dt][3];
    }
    if ((lane & 3) == 0) {
      sm[warp * 16 + rl] = m_lo;
      sm[warp * 16 + rh] = m_hi;
      sl[warp * 16 + rl] = l_lo;
      sl[warp * 16 + rh] = l_hi;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 16 * HD; e += 128) {
      const int r = e / HD, col = e % HD;
      const int m = cta_m0 + r;
      if (m >= M) continue;
      float mm = kNegBig;
#pragma unroll
      for (int w = 0; w < 4; ++w) mm = fmaxf(mm, sm[w * 16 + r]);
      float l = 0.f, acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = exp2f(sm[w * 16 + r] - mm);
        l += sl[w * 16 + r] * f;
        acc += so[(w * 16 + r) * HD + col] * f;
      }
      const int row = first + m / G, head = kvh * G + m % G;
      if (n_split == 1) {
        obuf[(static_cast<int64_t>(row) * n_q + head) * HD + col] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
      } else {
        part_o[((static_cast<int64_t>(sp) * rows_cap + row) * n_q + head) * HD + col] = acc;
        if (col == 0) part_ml[(static_cast<int64_t>(sp) * rows_cap + row) * n_q + head] = make_float2(mm, l);
      }
    }
  } else {
    const int rr[2] = {mlo, mhi};
    const float ll[2] = {l_lo, l_hi}, mmv[2] = {m_lo, m_hi};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = rr[h];
      if (m >= M) continue;
      const int row = first + m / G, head = kvh * G + m % G;
#pragma unroll
      for (int dt = 0; dt < kDT; ++dt) {
        const int col = dt * 8 + (lane & 3) * 2;
        const float a = o[dt][2 * h], b = o[dt][2 * h + 1];
        if (n_split == 1) {
          const float inv = ll[h] > 0.f ? 1.f / ll[h] : 0.f;
          *reinterpret_cast<__nv_bfloat162*>(obuf + (static_cast<int64_t>(row) * n_q + head) * HD + col) =
              __floats2bfloat162_rn(a * inv, b * inv);
        } else {
          float* po = part_o + ((static_cast<int64_t>(sp) * rows_cap + row) * n_q + head) * HD + col;
          po[0] = a;
          po[1] = b;
          if (dt == 0 && (lane & 3) == 0)
            part_ml[(static_cast<int64_t>(sp) * rows_cap + row) * n_q + head] = make_float2(mmv[h], ll[h]);
        }
      }
    }
  }
}

// One warp per (row, head): merge the KV-split partials.
template <int HD>
__global__ void attn_combine_kernel(RowsDev rows, int n_q, int n_split, int rows_cap,
                                    const float* __restrict__ part_o, const float2* __restrict__ part_ml,
                                    __nv_bfloat16* __restrict__ obuf) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int row = gw / n_q, head = gw % n_q;
  if (row >= *rows.n_rows) return;
  float mm = kNegBig;
  for (int s = 0; s < n_split; ++s) {
    mm = fmaxf(mm, part_ml[(static_cast<int64_t>(s) * rows_cap + row) * n_q + head].x);
  }
  float acc[HD / 32];
#pragma unroll
  for (int i = 0; i < HD / 32; ++i) acc[i] = 0.f;
  float l = 0.f;
  for (int s = 0; s < n_split; ++s) {
    const float2 ml = part_ml[(static_cast<int64_t>(s) * rows_cap + row) * n_q + head];
    const float f = exp2f(ml.x - mm);
    l += ml.y * f;
    const float* po = part_o + ((static_cast<int64_t>(s) * rows_cap + row) * n_q + head) * HD;
#pragma unroll
    for (int i = 0; i < HD / 32; ++i) acc[i] += po[lane + 32 * i] * f;
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
  for (int i = 0; i < HD / 32; ++i)
    obuf[(static_cast<int64_t>(row) * n_q + head) * HD + lane + 32 * i] = __float2bfloat16_rn(acc[i] * inv);
}

// Marks every split's (m, l) slot empty before the attention kernel runs, so splits that fall
// outside a request's causal range contribute nothing.
__global__ void attn_clear_ml_kernel(float2* ml, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ml[i] = make_float2(kNegBig, 0.f);
}

template <int HD, bool ROWS>
cudaError_t launch(const LlamaShape& m, RowsDev rows, int n_req, int blocks, int n_split, KvDev kv,
                   int layer, const __nv_bfloat16* qbuf, __nv_bfloat16* obuf, float* part_o,
                   float2* part_ml, int rows_cap, float scale_log2, cudaStream_t s) {
  constexpr int kTile = 64 * HD * 2;
  constexpr int kMerge = (4 * 16 * HD + 128) * 4;
  constexpr int kSmem = 4 * kTile > kMerge ? 4 * kTile : kMerge;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_kernel<HD, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = true;
  }
  dim3 grid(n_req, m.n_kv, blocks * n_split);
  attn_kernel<HD, ROWS><<<grid, 128, kSmem, s>>>(rows, kv, layer, m.n_q, m.n_kv, qbuf, obuf, part_o,
                                                 part_ml, n_split, rows_cap, scale_log2);
  return cudaGetLastError();
}

}  // namespace

cudaError_t lm_attention(const LlamaShape& m, RowsDev rows, int n_req, int max_rows_per_req,
                         int max_ctx, KvDev kv, int layer, const __nv_bfloat16* qbuf,
                         __nv_bfloat16* obuf, float* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (n_req <= 0 || max_rows_per_req <= 0) return cudaSuccess;
  if (m.hd != 64 && m.hd != 128) return cudaErrorInvalidValue;
  const int G = m.n_q / m.n_kv;
  const int Mmax = max_rows_per_req * G;
  const bool rows_mode = Mmax >= 64;
  const int blocks = rows_mode ? (Mmax + 63) / 64 : (Mmax + 15) / 16;
  const int rows_cap = n_req * max_rows_per_req;  // row indices are < sum of req_n <= this
  const int base = n_req * m.n_kv * blocks;
  const int tiles = (max_ctx + 63) / 64;
  int n_split = 1;
  if (base < 2 * 148 && tiles >= 4) {
    n_split = (2 * 148 + base - 1) / base;
    const int max_split = (tiles + 1) / 2;  // >= 2 pages per split
    if (n_split > max_split) n_split = max_split;
  }
  const size_t per_split = static_cast<size_t>(rows_cap) * m.n_q * (m.hd * 4 + 8);
  while (n_split > 1 && per_split * n_split > scratch_bytes) --n_split;
  float* part_o = scratch;
  float2* part_ml = reinterpret_cast<float2*>(scratch + static_cast<size_t>(n_split) * rows_cap * m.n_q * m.hd);
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(m.hd));
  // every (row, split) slot is written by its CTA (empty key ranges write (-1e30, 0)), so the
  // partial buffers need no clearing.
  cudaError_t e;
  if (m.hd == 64)
    e = rows_mode ? launch<64, true>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, rows_cap, scale_log2, s)
                  : launch<64, false>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, rows_cap, scale_log2, s);
  else
    e = rows_mode ? launch<128, true>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, rows_cap, scale_log2, s)
                  : launch<128, false>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, rows_cap, scale_log2, s);
  if (e != cudaSuccess || n_split == 1) return e;
  const int64_t warps = static_cast<int64_t>(rows_cap) * m.n_q;
  const int grid = static_cast<int>((warps * 32 + 255) / 256);
  if (m.hd == 64)
    attn_combine_kernel<64><<<grid, 256, 0, s>>>(rows, m.n_q, n_split, rows_cap, part_o, part_ml, obuf);
  else
    attn_combine_kernel<128><<<grid, 256, 0, s>>>(rows, m.n_q, n_split, rows_cap, part_o, part_ml, obuf);
  return cudaGetLastError();
}

}  // namespace faser

// tc_gemm.cu — tcgen05/TMEM GEMM for the draft and verification forwards (K1/K2).
//
//   ws[z][t][n] = sum_{k in split z} W[n][k] * X[t][k]        (bf16 x bf16 -> fp32)
//
// W is a weight matrix [N_out][K] (row-major = K-major), X the activations [T][K] of the
// ragged verify rows (T = sum k_i) or draft rows. The kernel is "swap-AB": the weights fill
// the 128-wide UMMA M dimension and the (few) tokens are the N dimension, so a verify batch
// of T = 5..256 rows is one N tile and the weights are streamed from HBM exactly once per
// split. Roles inside a 128-thread CTA:
//   warp 0 / lane 0 : TMA producer (W tile 128x64, X tile BNx64 per stage, SWIZZLE_128B)
//   warp 1 / lane 0 : tcgen05.mma issuer (UMMA 128xBNx16, accumulator in TMEM)
//   warp 2          : TMEM allocator
//   warps 0-3       : epilogue (tcgen05.ld 32 lanes x 16 columns -> fp32 partial tile)
// K is split across gridDim.z so that small-T launches still cover all 148 SMs; partial
// sums are reduced in a fixed order by the consumer kernel (deterministic, and independent
// of which rows survive early-exit pruning: the split count is fixed per forward).
// T can be read from device memory (t_dev) so that a forward whose row set shrinks on the
// device (early-exit compaction) launches once with its initial grid; tiles past the live
// row count exit immediately.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>

#include "sm100.cuh"
#include "tc_gemm.cuh"

namespace faser {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;                      // one 128-byte swizzle atom of bf16
constexpr int kUmmaK = 16;
constexpr int kABytes = kBM * kBK * 2;       // 16 KiB
constexpr int kXBox = 32;                    // activation TMA box rows

template <int BN>
struct Cfg {
  static constexpr int kStages = BN <= 32 ? 8 : BN <= 64 ? 7 : BN <= 128 ? 6 : 4;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kSmem = 1024 + kStages * kStageBytes + 256;
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   float* __restrict__ ws, int n_out, int t_stride, const int* __restrict__ t_dev,
                   int t_host, int kb_total, int kb_per_split) {
  using C = Cfg<BN>;
  const int T = t_dev ? min(*t_dev, t_host) : t_host;
  const int n0 = blockIdx.y * BN;
  if (n0 >= T) return;
  const int m0 = blockIdx.x * kBM;
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(kb_total, kb0 + kb_per_split);
  if (kb0 >= kb1) return;
  const int nkb = kb1 - kb0;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* accum = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::tma_prefetch(&tmW);
    sm100::tma_prefetch(&tmX);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(accum, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc<C::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------------------------------------------------------- TMA producer
    const uint64_t pol_w = sm100::policy_evict_first();
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      const uint32_t ph = (i / C::kStages) & 1;
      sm100::mbar_wait(&empty[s], ph ^ 1);
      sm100::mbar_arrive_expect_tx(&full[s], C::kStageBytes);
      const int kc = (kb0 + i) * kBK;
      sm100::tma_load_2d_hint(sA + s * kABytes, &tmW, &full[s], kc, m0, pol_w);
#pragma unroll
      for (int j = 0; j < (BN + kXBox - 1) / kXBox; ++j)
        sm100::tma_load_2d(sB + s * C::kBBytes + j * kXBox * 128, &tmX, &full[s], kc, n0 + j * kXBox);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      const uint32_t ph = (i / C::kStages) & 1;
      sm100::mbar_wait(&full[s], ph);
      sm100::tc_fence_after();
      const uint64_t da = sm100::desc_sw128(sm100::smem_u32(sA + s * kABytes));
      const uint64_t db = sm100::desc_sw128(sm100::smem_u32(sB + s * C::kBBytes));
#pragma unroll
      for (int k = 0; k < kBK / kUmmaK; ++k) {
        // advance along K inside the 128-byte swizzle atom: +32 bytes (>>4 = 2) per step
        sm100::mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
      }
      sm100::mma_commit(&empty[s]);
    }
    sm100::mma_commit(accum);
  }
  __syncwarp();

  // ------------------------------------------------------------------ epilogue
  sm100::mbar_wait(accum, 0);
  sm100::tc_fence_after();
  const int row = m0 + warp * 32 + lane;  // output feature of this thread
  float* out = ws + static_cast<size_t>(blockIdx.z) * t_stride * n_out;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    if (n0 + c0 >= T) break;
    float v[16];
    sm100::tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    if (row < n_out) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int t = n0 + c0 + i;
        if (t < T) out[static_cast<size_t>(t) * n_out + row] = v[i];
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) sm100::tmem_dealloc<C::kTmemCols>(tmem);
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

template <int BN>
void set_smem_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_tn_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmem);
  });
}

template <int BN>
cudaError_t launch_bn(const GemmOperand& w, const GemmOperand& x, float* ws, int t_stride,
                      const int* t_dev, int t, int splits, cudaStream_t s) {
  set_smem_attr<BN>();
  const int kb_total = w.k / kBK;
  const int kps = (kb_total + splits - 1) / splits;
  const int z = (kb_total + kps - 1) / kps;
  dim3 grid(w.rows / kBM, (t + BN - 1) / BN, z);
  gemm_tn_kernel<BN><<<grid, 128, Cfg<BN>::kSmem, s>>>(w.map, x.map, ws, w.rows, t_stride, t_dev, t,
                                                       kb_total, kps);
  return cudaGetLastError();
}

}  // namespace

cudaError_t make_operand(GemmOperand* op, const void* base, int rows, int k, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  if (k % kBK != 0) return cudaErrorInvalidValue;
  op->base = base;
  op->rows = rows;
  op->k = k;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(k) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&op->map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_weight_operand(GemmOperand* op, const void* w, int n_out, int k) {
  if (n_out % kBM != 0) return cudaErrorInvalidValue;
  return make_operand(op, w, n_out, k, kBM);
}
cudaError_t make_act_operand(GemmOperand* op, const void* x, int rows_cap, int k) {
  return make_operand(op, x, rows_cap, k, kXBox);
}

int gemm_bn_for(int t) { return t <= 32 ? 32 : t <= 64 ? 64 : t <= 128 ? 128 : 256; }

int gemm_splits_for(int n_out, int t, int k, int num_sms) {
  const int bn = gemm_bn_for(t);
  const int tiles = (n_out / kBM) * ((t + bn - 1) / bn);
  const int kb = k / kBK;
  int s = (num_sms + tiles - 1) / tiles;   // one wave of CTAs (1 CTA / SM)
  s = s < 1 ? 1 : s;
  const int max_s = kb / 4 > 0 ? kb / 4 : 1;  // >= 4 k-blocks (256 of K) per split
  return s > max_s ? max_s : s;
}

int gemm_effective_splits(int k, int splits) {
  const int kb = k / kBK;
  const int kps = (kb + splits - 1) / splits;
  return (kb + kps - 1) / kps;
}

cudaError_t gemm_tn(const GemmOperand& w, const GemmOperand& x, float* ws, int t_stride,
                    const int* t_dev, int t, int splits, cudaStream_t s) {
  if (t <= 0) return cudaSuccess;
  if (w.k != x.k) return cudaErrorInvalidValue;
  switch (gemm_bn_for(t)) {
    case 32: return launch_bn<32>(w, x, ws, t_stride, t_dev, t, splits, s);
    case 64: return launch_bn<64>(w, x, ws, t_stride, t_dev, t, splits, s);
    case 128: return launch_bn<128>(w, x, ws, t_stride, t_dev, t, splits, s);
    default: return launch_bn<256>(w, x, ws, t_stride, t_dev, t, splits, s);
  }
}

}  // namespace faser

// llama_attn_tc.cu — K3 on the 5th-generation tensor cores for GQA-packed verify / decode rows.
//
// One CTA per (request, kv head): the G query heads sharing the KV head are packed with the
// request's rows into the UMMA M dimension (m = row * G + g, M <= 64, padded to a 128-row tile;
// the padding rows are never read back). Per step of 128 keys (two 64-token pages):
//   S  = Q K^T      tcgen05.mma M128 x N128, K = head_dim; A = Q (smem, K-major SW128),
//                   B = the two K pages as TMA wrote them ([key][hd], K-major SW128); S in TMEM
//   softmax         4 warps, thread t = packed row t: its 128 scores come out of TMEM with
//                   tcgen05.ld (no shuffles), causal mask, running max / sum, the O rescale on
//                   TMEM (tcgen05.ld / st), P = exp2(S - m) as bf16 into smem (K-major SW128)
//   O += P V        tcgen05.mma M128 x N(head_dim), K = 128 keys; A = P, B = the two V pages
//                   read MN-major ([key][hd] rows = K, head_dim contiguous = N), O in TMEM
// Warp roles: warps 0-3 softmax / epilogue, warp 4 TMA producer (pages into a ring of steps),
// warp 5 MMA issuer. The epilogue divides O by the row sums and writes bf16 rows.
// Dispatch (llama_attn.cu, opt-in FASER_ATTN_TC=1): GROUP rows with G >= 4, M <= 64, no KV split,
// TMA view of the pool. Measured slower than the mma.sync kernel (see attn_tc_applies).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <mutex>

#include "llama.cuh"
#include "sm100.cuh"

namespace faser {
namespace {

constexpr float kNegBigT = -1e30f;
constexpr int kTcThreads = 192;     // 4 softmax warps + producer + MMA issuer
constexpr int kKeysPerStep = 128;   // two pages
constexpr int kMaxPagesTc = 512;

template <int HD>
struct TcCfg {
  static constexpr int kAtoms = HD / 64;                  // 128-byte swizzle atoms along head_dim
  static constexpr int kHalf = kKeysPerStep * 128;        // one atom column of a K or V step: 16 KB
  static constexpr int kStep = 2 * kAtoms * kHalf;        // K + V of one step
  static constexpr int kStages = HD == 64 ? 3 : 2;
  static constexpr int kQ = kAtoms * 128 * 128;           // Q tile [atom][128 rows][128 B]
  static constexpr int kP = 2 * 128 * 128;                // P tile [2 atoms of 64 keys][128 rows][128 B]
  static constexpr int kSmem = 1024 + kQ + kStages * kStep + kP;
  static constexpr uint32_t kTmemCols = 256;              // S [0, 128), O [128, 128 + HD)
};

__device__ __forceinline__ uint64_t desc_sw128_k(uint32_t saddr) { return sm100::desc_sw128(saddr); }
// MN-major SW128 operand: MN atoms of 64 elements (128 B) `lbo` bytes apart, K groups of 8 rows
// 1024 B apart (the [key][hd] page as TMA writes it, read with head_dim as N).
__device__ __forceinline__ uint64_t desc_sw128_mn(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
      "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
      "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
// 32 lanes x 32 columns without the completion wait (several loads share one tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int HD>
__global__ void __launch_bounds__(kTcThreads, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap kvmap, RowsDev rows,
                                                                 KvDev kv, int layer, int n_q, int n_kv,
                                                                 const __nv_bfloat16* __restrict__ qbuf,
                                                                 __nv_bfloat16* __restrict__ obuf, float scale_log2) {
  using C = TcCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = base;
  uint8_t* sKV = sQ + C::kQ;
  uint8_t* sP = sKV + C::kStages * C::kStep;
  __shared__ __align__(8) uint64_t full[C::kStages], empty[C::kStages];
  __shared__ __align__(8) uint64_t s_full, p_full, o_done;
  __shared__ uint32_t tmem_slot;
  __shared__ int s_page[kMaxPagesTc];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int req = blockIdx.x, kvh = blockIdx.y;
  const int nr = rows.req_n[req];
  const int gs = 31 - __clz(n_q / n_kv);
  const int G = 1 << gs, gm = G - 1;
  const int M = nr << gs;
  if (M == 0) return;
  const int first = rows.req_first[req], pos0 = rows.req_pos0[req], slot = rows.req_slot[req];
  const int key_end = pos0 + nr;  // keys [0, key_end)
  const int tiles = (key_end + 63) / 64;
  const int nsteps = (tiles + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  FASER_DCHECK(tiles <= kv.max_pages && tiles <= kMaxPagesTc, "FASER check: tc attention req %d pages %d\n", req, tiles);
  for (int i = threadIdx.x; i < tiles; i += kTcThreads) s_page[i] = kv.ptab[static_cast<int64_t>(slot) * kv.max_pages + i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(&s_full, 1);
    sm100::mbar_init(&p_full, 128);
    sm100::mbar_init(&o_done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0) sm100::tmem_alloc<C::kTmemCols>(&tmem_slot);
  // Q rows -> smem (K-major SW128): packed row m = r * G + g goes to tile row
  // t = (m % 4) * 32 + m / 4, so the <= 64 live rows spread over the four TMEM lane quarters
  // (one per softmax warp) instead of crowding the first
  for (int e = threadIdx.x; e < M * (HD / 8); e += kTcThreads) {
    const int m = e / (HD / 8), c = e % (HD / 8);
    const int t = ((m & 3) << 5) | (m >> 2);
    const uint4 v = *reinterpret_cast<const uint4*>(
        qbuf + (static_cast<int64_t>(first + (m >> gs)) * n_q + kvh * G + (m & gm)) * HD + c * 8);
    *reinterpret_cast<uint4*>(sQ + (c >> 3) * (128 * 128) + t * 128 + (((c & 7) ^ (t & 7)) << 4)) = v;
  }
  fence_proxy_async();  // generic smem writes (Q) visible to the tensor core (async proxy)
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 128;

  if (warp == 4) {
    // ---------------------------------------------------------------- TMA producer
    // one lane per TMA box (K/V x page x head_dim atom): a lane's boxes are served one after
    // another, so the step's 4 (hd 64) or 8 (hd 128) boxes are issued by as many lanes
    constexpr int kBoxes = 2 * 2 * C::kAtoms;
    if (lane < kBoxes) {
      const int64_t layer_rows = kv.layer_stride / HD;
      const int kvsel = lane & 1, p = (lane >> 1) & 1, h = lane >> 2;
      for (int u = 0; u < nsteps; ++u) {
        const int s = u % C::kStages;
        if (u >= C::kStages) sm100::mbar_wait(&empty[s], ((u / C::kStages) - 1) & 1);
        uint8_t* st = sKV + s * C::kStep;
        // a step past the last page re-loads it (finite data under the causal mask: P = 0 there)
        if (lane == 0) sm100::mbar_arrive_expect_tx(&full[s], kBoxes * 64 * 128);
        const int page = s_page[min(2 * u + p, tiles - 1)];
        FASER_DCHECK(static_cast<unsigned>(page) < kPageLimit, "FASER check: tc attention page %d\n", page);
        const int row = static_cast<int>(layer * layer_rows + (static_cast<int64_t>(page) * n_kv + kvh) * 2 * 64);
        // K: [atom h][key 64p .. 64p + 63][128 B]; V after all K atoms
        sm100::tma_load_2d(st + (kvsel * C::kAtoms + h) * C::kHalf + p * 64 * 128, &kvmap, &full[s], h * 64,
                           row + kvsel * 64);
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = sm100::idesc_bf16_f32(128, kKeysPerStep);
      constexpr uint32_t idesc_o = sm100::idesc_bf16_f32(128, HD) | (1u << 16);  // B (V) MN-major
      const uint32_t q0 = sm100::smem_u32(sQ), p0 = sm100::smem_u32(sP);
      for (int u = 0; u < nsteps; ++u) {
        const int s = u % C::kStages;
        sm100::mbar_wait(&full[s], (u / C::kStages) & 1);  // (softmax u-1 finished with S: p_full u-1)
        sm100::tc_fence_after();
        const uint32_t k0 = sm100::smem_u32(sKV + s * C::kStep);
        // S = Q K^T over head_dim (16 per instruction)
#pragma unroll
        for (int j = 0; j < HD / 16; ++j) {
          const uint64_t da = desc_sw128_k(q0 + (j >> 2) * (128 * 128)) + 2 * (j & 3);
          const uint64_t db = desc_sw128_k(k0 + (j >> 2) * C::kHalf) + 2 * (j & 3);
          sm100::mma_bf16(tS, da, db, idesc_s, j > 0 ? 1u : 0u);
        }
        sm100::mma_commit(&s_full);
        // O += P V over the step's 128 keys, once softmax u wrote P (and rescaled O)
        sm100::mbar_wait(&p_full, u & 1);
        sm100::tc_fence_after();
        const uint32_t v0 = k0 + C::kAtoms * C::kHalf;
#pragma unroll
        for (int j = 0; j < kKeysPerStep / 16; ++j) {
          const uint64_t da = desc_sw128_k(p0 + (j >> 2) * (128 * 128)) + 2 * (j & 3);
          const uint64_t db = desc_sw128_mn(v0 + j * 16 * 128, C::kHalf);  // 16 keys = 2 groups of 8 rows
          sm100::mma_bf16(tO, da, db, idesc_o, (u > 0 || j > 0) ? 1u : 0u);
        }
        sm100::mma_commit(&empty[s]);
        sm100::mma_commit(&o_done);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax + epilogue
    const int t = threadIdx.x;                  // tile row = TMEM lane
    const int m = ((t & 31) << 2) | (t >> 5);   // its packed row
    const int lim = m < M ? pos0 + (m >> gs) : -1;  // last key this row sees
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    float mrun = kNegBigT, lrun = 0.f;
    for (int u = 0; u < nsteps; ++u) {
      sm100::mbar_wait(&s_full, u & 1);
      sm100::tc_fence_after();
      const int kb = u * kKeysPerStep;
      uint32_t sr[kKeysPerStep];
#pragma unroll
      for (int c = 0; c < kKeysPerStep / 32; ++c)
        tmem_ld32_nw(tS + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_wait_ld();
      float mx = mrun;
#pragma unroll
      for (int i = 0; i < kKeysPerStep; ++i)
        if (kb + i <= lim) mx = fmaxf(mx, __uint_as_float(sr[i]) * scale_log2);
      const float alpha = exp2f(mrun - mx);
      // P(u) overwrites P(u-1): PV u-1 must have read it (and O must be final before the rescale)
      if (u > 0) {
        sm100::mbar_wait(&o_done, (u - 1) & 1);
        sm100::tc_fence_after();
      }
      // P = exp2(S - m) as bf16 into smem (K-major SW128: keys 0..63 atom 0, 64..127 atom 1)
      float sum = 0.f;
#pragma unroll
      for (int ch = 0; ch < kKeysPerStep / 8; ++ch) {
        float p8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int key = kb + ch * 8 + i;
          p8[i] = key <= lim ? exp2f(__uint_as_float(sr[ch * 8 + i]) * scale_log2 - mx) : 0.f;
          sum += p8[i];
        }
        uint4 pk;
        __nv_bfloat162 b0 = __floats2bfloat162_rn(p8[0], p8[1]), b1 = __floats2bfloat162_rn(p8[2], p8[3]);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(p8[4], p8[5]), b3 = __floats2bfloat162_rn(p8[6], p8[7]);
        pk.x = *reinterpret_cast<uint32_t*>(&b0);
        pk.y = *reinterpret_cast<uint32_t*>(&b1);
        pk.z = *reinterpret_cast<uint32_t*>(&b2);
        pk.w = *reinterpret_cast<uint32_t*>(&b3);
        *reinterpret_cast<uint4*>(sP + (ch >> 3) * (128 * 128) + t * 128 + (((ch & 7) ^ (t & 7)) << 4)) = pk;
      }
      lrun = lrun * alpha + sum;
      mrun = mx;
      // rescale the running O (PV u-1 has landed); tcgen05.ld/st are warp-collective, so the
      // warp skips only when none of its rows' max moved
      if (u > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        uint32_t orr[HD];
#pragma unroll
        for (int c = 0; c < HD / 32; ++c)
          tmem_ld32_nw(tO + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&orr[c * 32]));
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(orr[c * 32 + i]) * alpha;
          tmem_st32(tO + lane_off + c * 32, v);
        }
        tmem_wait_st();
      }
      fence_proxy_async();  // P (generic smem writes) visible to the tensor core
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full);
    }
    // ---- epilogue: O / l -> bf16 rows
    sm100::mbar_wait(&o_done, (nsteps - 1) & 1);
    sm100::tc_fence_after();
    const float inv = lrun > 0.f ? 1.f / lrun : 0.f;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      float v[32];
      sm100::tmem_ld32(tO + lane_off + c * 32, v);
      if (m < M) {
        __nv_bfloat16* od = obuf + (static_cast<int64_t>(first + (m >> gs)) * n_q + kvh * G + (m & gm)) * HD + c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 pk;
          __nv_bfloat162 b0 = __floats2bfloat162_rn(v[i] * inv, v[i + 1] * inv);
          __nv_bfloat162 b1 = __floats2bfloat162_rn(v[i + 2] * inv, v[i + 3] * inv);
          __nv_bfloat162 b2 = __floats2bfloat162_rn(v[i + 4] * inv, v[i + 5] * inv);
          __nv_bfloat162 b3 = __floats2bfloat162_rn(v[i + 6] * inv, v[i + 7] * inv);
          pk.x = *reinterpret_cast<uint32_t*>(&b0);
          pk.y = *reinterpret_cast<uint32_t*>(&b1);
          pk.z = *reinterpret_cast<uint32_t*>(&b2);
          pk.w = *reinterpret_cast<uint32_t*>(&b3);
          *reinterpret_cast<uint4*>(od + i) = pk;
        }
      }
    }
    sm100::tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<C::kTmemCols>(tmem);
  }
}

template <int HD>
cudaError_t launch_tc(const LlamaShape& m, RowsDev rows, int n_req, KvDev kv, int layer, const __nv_bfloat16* qbuf,
                      __nv_bfloat16* obuf, float scale_log2, cudaStream_t s) {
  using C = TcCfg<HD>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  dim3 grid(n_req, m.n_kv, 1);
  attn_tc_kernel<HD><<<grid, kTcThreads, C::kSmem, s>>>(*kv.tma, rows, kv, layer, m.n_q, m.n_kv, qbuf, obuf,
                                                       scale_log2);
  return cudaGetLastError();
}

}  // namespace

bool attn_tc_applies(const LlamaShape& m, int max_rows_per_req, int max_ctx, const KvDev& kv) {
  // opt-in (FASER_ATTN_TC=1): parity-green, but slower than the mma.sync kernel on B200 — the
  // per-step softmax over 128 keys runs on one warp per SM sub-partition (one 145-193 KB CTA
  // per SM) and is latency-bound at ~4 us per step (profiles/r02_attn_tc_ab.txt)
  static const bool on = getenv("FASER_ATTN_TC") && getenv("FASER_ATTN_TC")[0] == '1';
  const int G = m.n_q / m.n_kv;
  return on && kv.tma != nullptr && (m.hd == 64 || m.hd == 128) && G >= 4 && max_rows_per_req * G <= 64 &&
         (max_ctx + 63) / 64 <= kMaxPagesTc;
}

cudaError_t lm_attention_tc(const LlamaShape& m, RowsDev rows, int n_req, KvDev kv, int layer,
                            const __nv_bfloat16* qbuf, __nv_bfloat16* obuf, cudaStream_t s) {
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(m.hd));
  if (m.hd == 64) return launch_tc<64>(m, rows, n_req, kv, layer, qbuf, obuf, scale_log2, s);
  return launch_tc<128>(m, rows, n_req, kv, layer, qbuf, obuf, scale_log2, s);
}

}  // namespace faser

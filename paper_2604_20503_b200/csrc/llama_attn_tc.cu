// llama_attn_tc.cu — K3 on the 5th-generation tensor cores.
//
// One CTA per (request, kv head, 128-row tile): the G query heads sharing the KV head are packed
// with the request's rows into the UMMA M dimension (m = row * G + g, tiles of 128 packed rows;
// a request with <= 64 packed rows spreads them over all four softmax warps, padding rows are
// never read back). Per step of 128 keys (two 64-token pages):
//   S  = Q K^T      tcgen05.mma M128 x N128, K = head_dim; A = Q (smem, K-major SW128),
//                   B = the two K pages as TMA wrote them ([key][hd], K-major SW128); S in TMEM,
//                   double-buffered (S of step u+1 is issued before P V of step u)
//   softmax         8 warps: thread (quarter, half) owns tile row t and 64 of the step's keys,
//                   read out of TMEM with tcgen05.ld (no shuffles), the two halves' row maxima
//                   combined through smem; unmasked steps skip the causal compares; running
//                   max / sum on the raw scores (one FFMA + one MUFU.EX2 per key); the O rescale
//                   on TMEM is lazy (only when the max grew by 2^8); P = exp2(S - m) as bf16 into
//                   smem (K-major SW128, double-buffered for hd 64)
//   O += P V        tcgen05.mma M128 x N(head_dim), K = 128 keys; A = P, B = the two V pages
//                   read MN-major ([key][hd] rows = K, head_dim contiguous = N), O in TMEM
// Warp roles: warps 0-7 softmax / epilogue, warp 8 TMA producer (pages into a ring of steps),
// warp 9 MMA issuer. The epilogue divides O by the row sums and writes bf16 rows.
// Dispatch (llama_attn.cu): ROW blocks (> 64 packed rows per request: prefill, long verify) by
// default — about 2x the mma.sync kernel there; GQA-packed GROUP rows by default above 32 packed
// rows (where mma.sync reads each page twice); at <= 32 the one-CTA-per-SM footprint (512 TMEM
// columns, 145-193 KB smem) loses to mma.sync's occupancy (profiles/r02_attn_tc_ab.txt).
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
constexpr int kSmWarps = 8;         // softmax: 4 TMEM lane quarters x 2 key halves
constexpr int kTcThreads = (kSmWarps + 2) * 32;  // + TMA producer + MMA issuer
constexpr int kProdWarp = kSmWarps, kMmaWarp = kSmWarps + 1;
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
  static constexpr int kPBufs = HD == 64 ? 2 : 1;         // P double-buffered where smem allows
  static constexpr int kSmem = 1024 + kQ + kStages * kStep + kPBufs * kP;
  static constexpr uint32_t kTmemCols = 512;              // S0 [0,128), S1 [128,256), O [256, 256 + HD)
  static constexpr float kRescaleLog2 = 8.f;              // lazy O rescale once the max grows by 2^8
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
__device__ __forceinline__ float ex2(float x) {  // one MUFU.EX2
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int HD>
__global__ void __launch_bounds__(kTcThreads, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap kvmap, RowsDev rows,
                                                                 KvDev kv, int layer, int n_q, int n_kv,
                                                                 const __nv_bfloat16* __restrict__ qbuf,
                                                                 __nv_bfloat16* __restrict__ obuf, float scale_log2,
                                                                 int spread) {
  using C = TcCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (sm100::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = base;
  uint8_t* sKV = sQ + C::kQ;
  uint8_t* sP = sKV + C::kStages * C::kStep;
  __shared__ __align__(8) uint64_t full[C::kStages], empty[C::kStages];
  __shared__ __align__(8) uint64_t s_full[2], p_full[2], pv_done[2];  // by step parity
  __shared__ float xmax[2][2][128];  // [step parity][key half][tile row]: partial row maxima
  __shared__ float xsum[2][128];     // [key half][tile row]: partial row sums
  __shared__ uint32_t tmem_slot;
  __shared__ int s_page[kMaxPagesTc];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int req = blockIdx.x, kvh = blockIdx.y;
  const int nr = rows.req_n[req];
  const int gs = 31 - __clz(n_q / n_kv);
  const int G = 1 << gs, gm = G - 1;
  const int Mreq = nr << gs;
  const int m0 = blockIdx.z * 128;  // this CTA's 128 packed rows (prefill: several tiles per unit)
  if (m0 >= Mreq) return;
  const int M = min(128, Mreq - m0);  // live rows of the tile (tile-relative)
  const int first = rows.req_first[req], pos0 = rows.req_pos0[req], slot = rows.req_slot[req];
  const int key_end = pos0 + ((m0 + M - 1) >> gs) + 1;  // keys [0, key_end) for the tile's last row
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
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&s_full[b], 1);
      sm100::mbar_init(&p_full[b], kSmWarps * 32);
      sm100::mbar_init(&pv_done[b], 1);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 0) sm100::tmem_alloc<C::kTmemCols>(&tmem_slot);
  // Q rows -> smem (K-major SW128): tile row t holds packed row m0 + m (m = r * G + g). With
  // `spread` (<= 64 live rows) t = (m % 4) * 32 + m / 4, so the rows spread over the four TMEM
  // lane quarters (one per softmax warp) instead of crowding the first
  for (int e = threadIdx.x; e < M * (HD / 8); e += kTcThreads) {
    const int m = e / (HD / 8), c = e % (HD / 8);
    const int t = spread ? (((m & 3) << 5) | (m >> 2)) : m;
    const int mg = m0 + m;
    const uint4 v = *reinterpret_cast<const uint4*>(
        qbuf + (static_cast<int64_t>(first + (mg >> gs)) * n_q + kvh * G + (mg & gm)) * HD + c * 8);
    *reinterpret_cast<uint4*>(sQ + (c >> 3) * (128 * 128) + t * 128 + (((c & 7) ^ (t & 7)) << 4)) = v;
  }
  fence_proxy_async();  // generic smem writes (Q) visible to the tensor core (async proxy)
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t tO = tmem + 256;  // S(u) at tmem + (u % 2) * 128

  if (warp == kProdWarp) {
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
  } else if (warp == kMmaWarp) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = sm100::idesc_bf16_f32(128, kKeysPerStep);
      constexpr uint32_t idesc_o = sm100::idesc_bf16_f32(128, HD) | (1u << 16);  // B (V) MN-major
      const uint32_t q0 = sm100::smem_u32(sQ), p0 = sm100::smem_u32(sP);
      // S(u) is issued before PV(u-1), so the tensor core computes the next scores while the
      // softmax warps work on the current ones (S double-buffered in TMEM, P in smem)
      auto issue_s = [&](int u) {
        const int s = u % C::kStages;
        sm100::mbar_wait(&full[s], (u / C::kStages) & 1);
        sm100::tc_fence_after();
        const uint32_t k0 = sm100::smem_u32(sKV + s * C::kStep);
#pragma unroll
        for (int j = 0; j < HD / 16; ++j) {  // S = Q K^T over head_dim, 16 per instruction
          const uint64_t da = desc_sw128_k(q0 + (j >> 2) * (128 * 128)) + 2 * (j & 3);
          const uint64_t db = desc_sw128_k(k0 + (j >> 2) * C::kHalf) + 2 * (j & 3);
          sm100::mma_bf16(tmem + (u & 1) * 128, da, db, idesc_s, j > 0 ? 1u : 0u);
        }
        sm100::mma_commit(&s_full[u & 1]);
      };
      auto issue_pv = [&](int u) {  // O += P(u) V(u), once softmax u wrote P (and rescaled O)
        sm100::mbar_wait(&p_full[u & 1], (u >> 1) & 1);
        sm100::tc_fence_after();
        const int s = u % C::kStages;
        const uint32_t v0 = sm100::smem_u32(sKV + s * C::kStep) + C::kAtoms * C::kHalf;
        const uint32_t pb = p0 + (u % C::kPBufs) * C::kP;
#pragma unroll
        for (int j = 0; j < kKeysPerStep / 16; ++j) {
          const uint64_t da = desc_sw128_k(pb + (j >> 2) * (128 * 128)) + 2 * (j & 3);
          const uint64_t db = desc_sw128_mn(v0 + j * 16 * 128, C::kHalf);  // 16 keys = 2 groups of 8 rows
          sm100::mma_bf16(tO, da, db, idesc_o, (u > 0 || j > 0) ? 1u : 0u);
        }
        sm100::mma_commit(&empty[s]);
        sm100::mma_commit(&pv_done[u & 1]);
      };
      issue_s(0);
      for (int u = 1; u < nsteps; ++u) {
        issue_s(u);
        issue_pv(u - 1);
      }
      issue_pv(nsteps - 1);
    }
  } else {
    // ---------------------------------------------------------------- softmax + epilogue
    // warp w: TMEM lane quarter w % 4 (tile rows 32 (w % 4) ..), key half kh = w / 4 of each step
    // (64 keys, P atom kh, O columns [kh HD/2, (kh + 1) HD/2) for rescale and epilogue); the two
    // warps of a quarter combine their row maxima through smem at every step (named barrier)
    constexpr int kHalfKeys = kKeysPerStep / 2;
    const int qw = warp & 3, kh = warp >> 2;
    const int t = qw * 32 + lane;                             // tile row = TMEM lane
    const int m = spread ? (((t & 31) << 2) | (t >> 5)) : t;  // its tile-relative packed row
    const int mg = m0 + m;
    const int lim = m < M ? pos0 + (mg >> gs) : -1;           // last key this row sees
    const uint32_t lane_off = static_cast<uint32_t>(qw * 32) << 16;
    const uint32_t ocol = kh * (HD / 2);
    auto pair_sync = [&] { asm volatile("bar.sync %0, 64;" ::"r"(1 + qw) : "memory"); };
    // warp-uniform: the smallest causal limit among the warp's live rows (steps entirely below it
    // need no masking; padded rows compute garbage that only their own, never-written rows see)
    const int wlim = __reduce_min_sync(0xffffffffu, m < M ? lim : 0x7fffffff);
    float mused = kNegBigT, lrun = 0.f;  // reference max of P and O (lazily raised), partial row sum
    for (int u = 0; u < nsteps; ++u) {
      sm100::mbar_wait(&s_full[u & 1], (u >> 1) & 1);
      sm100::tc_fence_after();
      const int kb = u * kKeysPerStep + kh * kHalfKeys;
      uint32_t sr[kHalfKeys];
#pragma unroll
      for (int c = 0; c < kHalfKeys / 32; ++c)
        tmem_ld32_nw(tmem + (u & 1) * 128 + kh * kHalfKeys + lane_off + c * 32,
                     *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_wait_ld();
      const bool full_step = kb + kHalfKeys - 1 <= wlim;  // no key of this half is masked
      float mx4[4] = {kNegBigT, kNegBigT, kNegBigT, kNegBigT};  // independent chains, raw scores
      if (full_step) {
#pragma unroll
        for (int i = 0; i < kHalfKeys; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(sr[i]));
      } else {
#pragma unroll
        for (int i = 0; i < kHalfKeys; ++i)
          if (kb + i <= lim) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(sr[i]));
      }
      xmax[u & 1][kh][t] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      pair_sync();
      const float mraw = fmaxf(xmax[u & 1][0][t], xmax[u & 1][1][t]);  // same value in both halves
      const float mx = mraw > kNegBigT ? mraw * scale_log2 : kNegBigT;  // (scale > 0)
      if (u == 0) {
        mused = mx;
      } else if (__any_sync(0xffffffffu, mx > mused + C::kRescaleLog2)) {
        // the quarter raises its reference max (both halves decide alike): O must be current (PV
        // u-1 landed) to rescale it; each half rescales its O columns
        sm100::mbar_wait(&pv_done[(u - 1) & 1], ((u - 1) >> 1) & 1);
        sm100::tc_fence_after();
        const float mnew = fmaxf(mused, mx);
        const float alpha = exp2f(mused - mnew);
        uint32_t orr[HD / 2];
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tmem_ld32_nw(tO + ocol + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&orr[c * 32]));
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(orr[c * 32 + i]) * alpha;
          tmem_st32(tO + ocol + lane_off + c * 32, v);
        }
        tmem_wait_st();
        lrun *= alpha;
        mused = mnew;
      }
      // P(u) reuses the buffer PV(u - kPBufs) read
      if (u >= C::kPBufs) {
        const int w = u - C::kPBufs;
        sm100::mbar_wait(&pv_done[w & 1], (w >> 1) & 1);
      }
      // P = exp2(S - m_ref) as bf16 (K-major SW128: this half's 64 keys are P atom kh)
      uint8_t* pbuf = sP + (u % C::kPBufs) * C::kP + kh * (128 * 128);
      float sum4[4] = {0.f, 0.f, 0.f, 0.f};
      const float nm = -mused;
#pragma unroll
      for (int ch = 0; ch < kHalfKeys / 8; ++ch) {
        float p8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float e = ex2(fmaf(__uint_as_float(sr[ch * 8 + i]), scale_log2, nm));
          p8[i] = (full_step || kb + ch * 8 + i <= lim) ? e : 0.f;
          sum4[i & 3] += p8[i];
        }
        uint4 pk;
        __nv_bfloat162 b0 = __floats2bfloat162_rn(p8[0], p8[1]), b1 = __floats2bfloat162_rn(p8[2], p8[3]);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(p8[4], p8[5]), b3 = __floats2bfloat162_rn(p8[6], p8[7]);
        pk.x = *reinterpret_cast<uint32_t*>(&b0);
        pk.y = *reinterpret_cast<uint32_t*>(&b1);
        pk.z = *reinterpret_cast<uint32_t*>(&b2);
        pk.w = *reinterpret_cast<uint32_t*>(&b3);
        *reinterpret_cast<uint4*>(pbuf + t * 128 + ((ch ^ (t & 7)) << 4)) = pk;
      }
      lrun += (sum4[0] + sum4[1]) + (sum4[2] + sum4[3]);
      fence_proxy_async();  // P (generic smem writes) visible to the tensor core
      sm100::tc_fence_before();
      sm100::mbar_arrive(&p_full[u & 1]);
    }
    // ---- epilogue: O / l -> bf16 rows (each half its O columns; l = both halves' sums)
    xsum[kh][t] = lrun;
    pair_sync();
    const float l = xsum[0][t] + xsum[1][t];
    sm100::mbar_wait(&pv_done[(nsteps - 1) & 1], ((nsteps - 1) >> 1) & 1);
    sm100::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int c = 0; c < HD / 64; ++c) {
      float v[32];
      sm100::tmem_ld32(tO + ocol + lane_off + c * 32, v);
      if (m < M) {
        __nv_bfloat16* od =
            obuf + (static_cast<int64_t>(first + (mg >> gs)) * n_q + kvh * G + (mg & gm)) * HD + ocol + c * 32;
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
cudaError_t launch_tc(const LlamaShape& m, RowsDev rows, int n_req, int max_rows_per_req, KvDev kv, int layer,
                      const __nv_bfloat16* qbuf, __nv_bfloat16* obuf, float scale_log2, cudaStream_t s) {
  using C = TcCfg<HD>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  const int Mmax = max_rows_per_req * (m.n_q / m.n_kv);
  dim3 grid(n_req, m.n_kv, (Mmax + 127) / 128);
  attn_tc_kernel<HD><<<grid, kTcThreads, C::kSmem, s>>>(*kv.tma, rows, kv, layer, m.n_q, m.n_kv, qbuf, obuf,
                                                       scale_log2, Mmax <= 64 ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace

bool attn_tc_rows_applies(const LlamaShape& m, int max_ctx, const KvDev& kv) {
  // prefill / long-row blocks (> 64 packed rows): 128-row tiles keep all four softmax warps busy
  // (FASER_ATTN_TC_ROWS=0 keeps the mma.sync ROWS kernel)
  static const bool on = !(getenv("FASER_ATTN_TC_ROWS") && getenv("FASER_ATTN_TC_ROWS")[0] == '0');
  return on && kv.tma != nullptr && (m.hd == 64 || m.hd == 128) && (max_ctx + 63) / 64 <= kMaxPagesTc;
}

bool attn_tc_applies(const LlamaShape& m, int max_rows_per_req, int max_ctx, const KvDev& kv) {
  // GQA-packed GROUP rows: by default only above 32 packed rows, where the mma.sync kernel needs
  // two 32-row blocks per (request, kv head) and so reads the KV pages twice; at <= 32 rows it keeps
  // several CTAs per SM and wins (one CTA per SM here: 512 TMEM columns). FASER_ATTN_TC=1 takes
  // every GROUP shape, =0 none (profiles/r02_attn_tc_ab.txt, r02_attn_group_split.txt)
  static const char* env = getenv("FASER_ATTN_TC");
  static const int force = env ? (env[0] == '1' ? 1 : 0) : -1;
  const int G = m.n_q / m.n_kv;
  const bool shape = kv.tma != nullptr && (m.hd == 64 || m.hd == 128) && G >= 4 && max_rows_per_req * G <= 64 &&
                     (max_ctx + 63) / 64 <= kMaxPagesTc;
  return shape && (force == 1 || (force < 0 && max_rows_per_req * G > 32));
}

cudaError_t lm_attention_tc(const LlamaShape& m, RowsDev rows, int n_req, int max_rows_per_req, KvDev kv, int layer,
                            const __nv_bfloat16* qbuf, __nv_bfloat16* obuf, cudaStream_t s) {
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(m.hd));
  if (m.hd == 64) return launch_tc<64>(m, rows, n_req, max_rows_per_req, kv, layer, qbuf, obuf, scale_log2, s);
  return launch_tc<128>(m, rows, n_req, max_rows_per_req, kv, layer, qbuf, obuf, scale_log2, s);
}

}  // namespace faser

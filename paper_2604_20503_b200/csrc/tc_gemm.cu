// tc_gemm.cu — tcgen05/TMEM GEMM with fused split-K reduction and row epilogues, the
// projection engine of the draft (K1) and verification (K2) forwards.
//
//   D[n][t] = sum_k W[n][k] * X[t][k]           (bf16 x bf16 -> fp32 in TMEM)
//
// "Swap-AB": the weights fill the 128-wide UMMA M dimension and the verify/draft rows are the
// N dimension, so a batch of T = 1..256 rows is one N tile and the weights stream from HBM
// exactly once. Roles in a 128-thread CTA:
//   warp 0          : TMA producers, one lane group per pipeline stage (W tiles 128x64 x MC,
//                     X tile BNx64 per stage, SWIZZLE_128B)
//   warp 1 / lane 0 : tcgen05.mma issuer (UMMA 128xBNx16), commits free smem stages
//   warp 2          : TMEM allocator
//   warps 2-3       : per-token prologue (RMSNorm scale, positions, KV pages) during the mainloop
//   warps 0-3       : epilogue
// K is split over gridDim.z so small-T launches cover all SMs; the split CTAs of a tile are one
// thread-block cluster and reduce their fp32 partials through DSMEM in rank order (deterministic,
// independent of which rows survive early-exit pruning because the split count is fixed per
// forward), each CTA then runs the fused epilogue on its slice of the tile's tokens:
//   store | residual add (+ per-tile sum of squares for the next RMSNorm) | RoPE + q write +
//   paged KV append | SwiGLU | logits (+ per-tile argmax).
// RMSNorm is folded: the GEMM consumes the un-normalised residual (bf16) and scales each token
// column by rsqrt(mean(x^2)+eps) in the epilogue (W.(x*r) = r*(W.x)); gamma = 1 for these
// random-init models.
// Launch uses programmatic dependent launch: the prologue (barrier init, TMEM alloc, tensor-map
// prefetch) overlaps the previous kernel; every dependent read is after griddepcontrol.wait.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <utility>
#include <cmath>
#include <unordered_map>

#include "sm100.cuh"
#include "tc_gemm.cuh"

namespace faser {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;                      // one 128-byte swizzle atom of bf16
constexpr int kUmmaK = 16;
constexpr int kABytes = kBM * kBK * 2;       // 16 KiB
constexpr int kXBox = 32;                    // activation TMA box rows

// ST = pipeline depth: "shallow" 4-stage configs (~100 KB smem for BN <= 64, 2 CTAs / SM, room
// for the next GEMM's weight prefetch) or "deep" configs filling ~200 KB (1 CTA / SM).
// MC = weight tiles (of 128 rows) per CTA sharing one rows tile: each SM's TMA ingest (~44 GB/s
// per SM on B200, tools/tma_probe.cu) is spent on MC weight blocks per rows block instead of one.
template <int BN, int ST, int MC>
struct Cfg {
  static constexpr int kStages = ST;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kAStage = MC * kABytes;
  static constexpr int kStageBytes = kAStage + kBBytes;
  static constexpr int kTmemNeed = MC * (BN < 32 ? 32 : BN);
  static constexpr int kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128 : kTmemNeed <= 256 ? 256 : 512;
  static constexpr int kPipe = kStages * kStageBytes;
  static constexpr int kTile = BN * kBM * 4;  // fp32 epilogue staging tile (one weight tile at a time)
  static constexpr int kSmem = 1024 + (kPipe > kTile ? kPipe : kTile) + 12288;
};

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t map_cta(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp(const EpiArgs& ea, int i) {
  if (ea.trace) {
    const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    ea.trace[cta * 8 + i] = gtimer();
  }
}
// Coupled Gumbel-max sampling noise (faser_set_sampling). The draft and the target perturb the
// logits that predict absolute position `pos` of request `rid` with the SAME noise, so a drafted
// token is accepted iff it equals the target's own sample: every committed token is the target's
// Gumbel-max sample of softmax(z / tau) given its prefix (lossless in distribution, and identical
// to non-speculative sampling with this noise whatever the drafter proposes). SplitMix64 mixing;
// u = (23 random bits + 0.5) * 2^-23 in (0, 1) exactly, g = -log(-log(u)) in fp32.
__device__ __forceinline__ uint64_t smix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t sample_key(uint64_t seed, int64_t rid, int pos) {
  return smix64(smix64(seed) ^ (static_cast<uint64_t>(rid) * 0xd1b54a32d192ed03ull) ^
                (static_cast<uint64_t>(pos) * 0x8cb92ba72f3d8dd7ull));
}
__device__ __forceinline__ float gumbel(uint64_t key, int id) {
  const uint64_t h = smix64(key ^ (static_cast<uint64_t>(id) * 0x9e3779b97f4a7c15ull));
  const float u = (static_cast<float>(static_cast<uint32_t>(h >> 41)) + 0.5f) * 0x1p-23f;
  return -logf(-logf(u));
}
__device__ __forceinline__ float perturb(float z, float inv_tau, uint64_t key, int id) {
  return __fadd_rn(__fmul_rn(z, inv_tau), gumbel(key, id));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <int BN, int ST, int MC>
__global__ void __launch_bounds__(128, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ EpiArgs ea, int n_out, int kb_total, int kb_per_split, int splits,
                int issue, int xbox) {
  using C = Cfg<BN, ST, MC>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kAStage;
  uint8_t* aux = smem + (C::kPipe > C::kTile ? C::kPipe : C::kTile);
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + C::kStages;
  uint64_t* accum = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  float* s_rs = reinterpret_cast<float*>(aux + 256);  // [256] per-token RMSNorm scale
  float* s_red = s_rs + 256;                          // [4][BN] per-warp partials
  int* s_i0 = reinterpret_cast<int*>(s_red + 4 * 256);  // [4][BN] per-warp argmax ids
  int* s_pos = s_i0 + 4 * 256;  // [256] per-token position (QKV epilogue)
  int* s_page = s_pos + 256;    // [256] per-token KV page
  uint64_t* s_key = reinterpret_cast<uint64_t*>(s_red);  // [256] sampling keys (kEpiLogits / kEpiRank)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mb = blockIdx.x * MC * kBM;                       // first weight row of this CTA
  const int ntile = min(MC, n_out / kBM - static_cast<int>(blockIdx.x) * MC);  // weight tiles here
  const int n0 = ea.t_begin + blockIdx.y * BN;
  const int kb0 = blockIdx.z * kb_per_split;
  const int kb1 = min(kb_total, kb0 + kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    stamp(ea, 0);
    sm100::tma_prefetch(&tmW);
    sm100::tma_prefetch(&tmX);
    for (int s = 0; s < C::kStages; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    sm100::mbar_init(accum, 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();  // barrier inits visible before the producer touches them
  pdl_trigger();
  // Weights do not depend on the previous kernel: stream the first stages of this CTA's weight
  // slice now, overlapping the previous kernel's tail (programmatic dependent launch).
  //
  // TMA issue is spread over the producer warp: B200's TMA serves the box requests of one issuing
  // thread one after another (tools/tma_probe.cu: one thread ~40 GB/s per SM, four threads
  // ~105-160 GB/s). `issue` = ngrp * 100 + gsz: ngrp lane groups (1, or one per stage: a stage is
  // only ever filled by one group, so the empty/full parity protocol is the single-producer one),
  // gsz lanes per group splitting the stage's boxes. The group's leader (g == 0) owns the stage's
  // mbarrier accounting (expect_tx for all of the stage's bytes, before its own arrive); the other
  // lanes only issue boxes, whose complete_tx may land before the leader's expect_tx (tx-count may
  // go transiently negative; the phase cannot complete before the arrive).
  const int ngrp = issue / 100, gsz = issue % 100;
  const int pst = lane / gsz, pg = lane % gsz;  // lane group (first stage) and box slot of this lane
  const bool producer = warp == 0 && pst < ngrp;
  const int npre = ea.w_after_wait ? 0 : (nkb < C::kStages ? nkb : C::kStages);
  const uint64_t pol_w = sm100::policy_evict_first();
  if (producer) {
    for (int i = pst; i < npre; i += ngrp) {
      if (pg == 0) sm100::mbar_expect_tx(&full[i], ntile * kABytes);
      for (int j = pg; j < ntile; j += gsz)
        sm100::tma_load_2d_hint(sA + i * C::kAStage + j * kABytes, &tmW, &full[i], (kb0 + i) * kBK, mb + j * kBM, pol_w);
    }
  }
  pdl_wait();  // everything below may read the previous kernel's output
  if (threadIdx.x == 0) stamp(ea, 1);
  const int T = ea.n_rows ? min(*ea.n_rows, ea.t_stride) : ea.t_stride;
  if (n0 >= T) {  // uniform per CTA: tile entirely past the live rows (early-exit compaction)
    if (producer && pg == 0) {  // drain the prefetched weight tiles before exiting
      for (int i = pst; i < npre; i += ngrp) sm100::mbar_arrive(&full[i]);
      for (int i = pst; i < npre; i += ngrp) sm100::mbar_wait(&full[i], 0);
    }
    return;
  }
  if (warp == 2) sm100::tmem_alloc<C::kTmemCols>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producers (one lane group per stage)
    const int xboxes = (min(BN, T - n0) + xbox - 1) / xbox;  // skip all-padding activation boxes
    const uint32_t xbytes = xboxes * xbox * kBK * 2;
    if (producer) {
      for (int i = pst; i < nkb; i += ngrp) {
        const int s = i % C::kStages;
        const uint32_t ph = (i / C::kStages) & 1;
        const int kc = (kb0 + i) * kBK;
        const bool pre = i < npre;  // weight tiles already in flight from the prologue
        if (!pre) sm100::mbar_wait(&empty[s], ph ^ 1);
        if (pg == 0) sm100::mbar_arrive_expect_tx(&full[s], (pre ? 0 : ntile * kABytes) + xbytes);
        const int nw = pre ? 0 : ntile;  // boxes of this stage: nw weight boxes, then xboxes rows boxes
        for (int b = pg; b < nw + xboxes; b += gsz) {
          if (b < nw)
            sm100::tma_load_2d_hint(sA + s * C::kAStage + b * kABytes, &tmW, &full[s], kc, mb + b * kBM, pol_w);
          else
            sm100::tma_load_2d(sB + s * C::kBBytes + (b - nw) * xbox * 128, &tmX, &full[s], kc, n0 + (b - nw) * xbox);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = sm100::idesc_bf16_f32(kBM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      const uint32_t ph = (i / C::kStages) & 1;
      sm100::mbar_wait(&full[s], ph);
      sm100::tc_fence_after();
      if (i == 0) stamp(ea, 2);
      const uint64_t db = sm100::desc_sw128(sm100::smem_u32(sB + s * C::kBBytes));
      for (int j = 0; j < ntile; ++j) {  // every weight tile of the stage against the same rows tile
        const uint64_t da = sm100::desc_sw128(sm100::smem_u32(sA + s * C::kAStage + j * kABytes));
#pragma unroll
        for (int k = 0; k < kBK / kUmmaK; ++k)  // +32 bytes along K inside the swizzle atom
          sm100::mma_bf16(tmem + j * (BN < 32 ? 32 : BN), da + 2 * k, db + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
      }
      sm100::mma_commit(&empty[s]);
    }
    sm100::mma_commit(accum);
  } else if (warp >= 2) {
    // Per-token prologue, computed by the two otherwise idle warps while the mainloop streams:
    // RMSNorm scale of the un-normalised residual input and, for the QKV epilogue, the token's
    // position and KV page (a dependent load chain that would otherwise sit after the MMAs).
    const int tn0 = min(BN, T - n0);
    for (int t = threadIdx.x - 64; t < tn0; t += 64) {
      float rs = 1.f;
      if (ea.ss_in) {
        float part[4] = {0.f, 0.f, 0.f, 0.f};
        for (int c = 0; c < ea.ss_chunks; c += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c + u < ea.ss_chunks) part[u] += ea.ss_in[static_cast<size_t>(c + u) * ea.t_stride + n0 + t];
        }
        rs = rsqrtf(((part[0] + part[1]) + (part[2] + part[3])) / ea.d_norm + ea.eps);
      }
      s_rs[t] = rs;
      if ((ea.mode == kEpiLogits || ea.mode == kEpiRank) && ea.inv_tau > 0.f) {  // the row's sampling key
        const int row = n0 + t;
        s_key[t] = sample_key(ea.samp_seed, ea.req_ids[ea.rows.row_req[row]], ea.rows.row_pos[row] + 1);
      }
      if (ea.mode == kEpiRank) {  // the row's drafted id and its z_d (s_pos / s_page reused)
        const int row = n0 + t;
        const int dd = ea.row_d[row];
        float zd = ea.zd_src[static_cast<size_t>(row) * kBM + (row & (kBM - 1))];
        // sampling: rank d among the perturbed values, its own perturbed the same way
        if (ea.inv_tau > 0.f && dd >= 0) zd = perturb(zd, ea.inv_tau, s_key[t], dd);
        s_pos[t] = dd;
        s_page[t] = __float_as_int(zd);
      }
      if (ea.mode == kEpiQkv) {
        const int row = n0 + t;
        const int pos = ea.rows.row_pos[row];
        const int slot = ea.rows.req_slot[ea.rows.row_req[row]];
        s_pos[t] = pos;
        s_page[t] = ea.kv.ptab[static_cast<size_t>(slot) * ea.kv.max_pages + pos / kPage];
        FASER_DCHECK(pos >= 0 && pos / kPage < ea.kv.max_pages && static_cast<unsigned>(s_page[t]) < kPageLimit,
                     "FASER check: qkv epilogue row %d slot %d pos %d page %d\n", row, slot, pos, s_page[t]);
      }
    }
  }
  __syncwarp();

  // ------------------------------------------------------------------ epilogue
  sm100::mbar_wait(accum, 0);
  sm100::tc_fence_after();
  if (threadIdx.x == 0) stamp(ea, 3);
  const int tn = min(BN, T - n0);          // live tokens of this tile
#pragma unroll 1
  for (int j = 0; j < ntile; ++j) {        // weight tiles of this CTA, one staging pass each
  const int m0 = mb + j * kBM;
    const int r = warp * 32 + lane;          // tile row owned in the TMEM read-out
    float* S = reinterpret_cast<float*>(smem);  // [BN][128] fp32 staging (pipeline smem is free now)
  #pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      if (c0 >= tn) break;
      float v[32];
      sm100::tmem_ld32(tmem + j * (BN < 32 ? 32 : BN) + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);  // one wait per 32 columns
  #pragma unroll
      for (int i = 0; i < 32; ++i) S[(c0 + i) * kBM + r] = v[i];
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 2 && j == ntile - 1) sm100::tmem_dealloc<C::kTmemCols>(tmem);
    // Split-K: the `splits` CTAs of this tile are one thread-block cluster. Each owns a slice of the
    // tile's tokens and sums that slice over every CTA's partial through DSMEM in rank order
    // (deterministic), then runs the epilogue on its slice.
    int ts = 0, te = tn;
    if (splits > 1) {
      cluster_sync();
      if (threadIdx.x == 0 && j == 0) stamp(ea, 6);
      const int per = (tn + splits - 1) / splits;
      ts = min(tn, static_cast<int>(blockIdx.z) * per);
      te = min(tn, ts + per);
      const uint32_t base = sm100::smem_u32(S);
      uint32_t rb[16];
  #pragma unroll
      for (int z = 0; z < 16; ++z) rb[z] = z < splits ? map_cta(base, z) : 0u;
      const int c4 = threadIdx.x & 31, tq = threadIdx.x >> 5;  // 4 rows (float4) x 4 tokens per pass
      // two passes per round: every DSMEM load of the round is issued before any sum or store
      // (one remote latency per round instead of one per pass); sums stay in rank order
      for (int t = ts + tq; t < te; t += 8) {
        const int t2 = t + 4;
        const bool two = t2 < te;
        float4 v[2][16];
  #pragma unroll
        for (int z = 0; z < 16; ++z) {
          if (z < splits) {
            v[0][z] = ld_dsmem4(rb[z] + (t * kBM + c4 * 4) * 4);
            if (two) v[1][z] = ld_dsmem4(rb[z] + (t2 * kBM + c4 * 4) * 4);
          }
        }
  #pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  #pragma unroll
          for (int z = 0; z < 16; ++z) {
            if (z < splits) {
              a.x += v[h][z].x;
              a.y += v[h][z].y;
              a.z += v[h][z].z;
              a.w += v[h][z].w;
            }
          }
          // only this CTA reads its own slice rows, so the in-place write is race-free
          *reinterpret_cast<float4*>(S + (h ? t2 : t) * kBM + c4 * 4) = a;
        }
      }
      // done reading the peers' partials: let them proceed (their exit / next tile waits only
      // for this arrive), while this CTA runs its epilogue
      cluster_arrive();
      __syncthreads();
    }
    __syncthreads();  // (the per-token prologue was written by warps 2-3 during the mainloop)
    if (threadIdx.x == 0 && j == 0) stamp(ea, 4);

    // Token-per-warp passes: lane owns 4 consecutive tile rows (float4), a warp covers the 128
    // rows of one token, 4 tokens per pass.
    const int mode = ea.mode;
    const int c4 = lane * 4;
    if (mode == kEpiStore || mode == kEpiResid || mode == kEpiLogits || mode == kEpiRank) {
      for (int t = ts + warp; t < te; t += 4) {
        const float rs = s_rs[t];
        float4 a = *reinterpret_cast<const float4*>(S + t * kBM + c4);
        const size_t idx = static_cast<size_t>(n0 + t) * n_out + m0 + c4;
        if (mode == kEpiStore) {
          if (ea.out_bf16) {
            __nv_bfloat162 b0 = __floats2bfloat162_rn(a.x * rs, a.y * rs), b1 = __floats2bfloat162_rn(a.z * rs, a.w * rs);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&b0);
            pk.y = *reinterpret_cast<uint32_t*>(&b1);
            *reinterpret_cast<uint2*>(ea.out_bf16 + idx) = pk;
          } else {
            *reinterpret_cast<float4*>(ea.out + idx) = make_float4(a.x * rs, a.y * rs, a.z * rs, a.w * rs);
          }
        } else if (mode == kEpiResid) {
          const float4 xv = *reinterpret_cast<const float4*>(ea.x + idx);
          a = make_float4(xv.x + a.x, xv.y + a.y, xv.z + a.z, xv.w + a.w);
          *reinterpret_cast<float4*>(ea.x + idx) = a;
          __nv_bfloat162 b0 = __floats2bfloat162_rn(a.x, a.y), b1 = __floats2bfloat162_rn(a.z, a.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&b0);
          pk.y = *reinterpret_cast<uint32_t*>(&b1);
          *reinterpret_cast<uint2*>(ea.xb + idx) = pk;
          float q = (a.x * a.x + a.y * a.y) + (a.z * a.z + a.w * a.w);
  #pragma unroll
          for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
          if (lane == 0) ea.ss_out[static_cast<size_t>(m0 / kBM) * ea.t_stride + n0 + t] = q;
        } else if (mode == kEpiRank) {
          // token_exit_test's rank count (exitctl.cpp:56-68) on this tile's 128 ids: the same
          // fp32 products acc * rs as the materialised logits, compared against z_d
          a = make_float4(a.x * rs, a.y * rs, a.z * rs, a.w * rs);
          if (ea.logits) *reinterpret_cast<float4*>(ea.logits + idx) = a;  // debug capture only
          const float zd = __int_as_float(s_page[t]);
          const int dd = s_pos[t];
          const int id0 = ea.id_off + m0 + c4;
          if (ea.inv_tau > 0.f) {  // sampling: the exit test ranks the perturbed values
            const uint64_t key = s_key[t];
            a = make_float4(perturb(a.x, ea.inv_tau, key, id0), perturb(a.y, ea.inv_tau, key, id0 + 1),
                            perturb(a.z, ea.inv_tau, key, id0 + 2), perturb(a.w, ea.inv_tau, key, id0 + 3));
          }
          int c = 0;
          c += (id0 != dd) & ((a.x > zd) | ((a.x == zd) & (id0 < dd)));
          c += (id0 + 1 != dd) & ((a.y > zd) | ((a.y == zd) & (id0 + 1 < dd)));
          c += (id0 + 2 != dd) & ((a.z > zd) | ((a.z == zd) & (id0 + 2 < dd)));
          c += (id0 + 3 != dd) & ((a.w > zd) | ((a.w == zd) & (id0 + 3 < dd)));
  #pragma unroll
          for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
          if (lane == 0) ea.rank_cnt[static_cast<size_t>(m0 / kBM) * ea.t_stride + n0 + t] = c;
        } else {  // kEpiLogits
          a = make_float4(a.x * rs, a.y * rs, a.z * rs, a.w * rs);
          if (ea.logits) *reinterpret_cast<float4*>(ea.logits + idx) = a;  // validation / exit test only
          const int id0 = ea.id_off + m0 + c4;
          if (ea.inv_tau > 0.f) {  // Gumbel-max sampling: argmax of z / tau + g
            const uint64_t key = s_key[t];
            a = make_float4(perturb(a.x, ea.inv_tau, key, id0), perturb(a.y, ea.inv_tau, key, id0 + 1),
                            perturb(a.z, ea.inv_tau, key, id0 + 2), perturb(a.w, ea.inv_tau, key, id0 + 3));
          }
          if (ea.id_limit && id0 + 3 >= ea.id_limit) {  // vocab padding of a TP shard
            if (id0 >= ea.id_limit) a.x = -FLT_MAX;
            if (id0 + 1 >= ea.id_limit) a.y = -FLT_MAX;
            if (id0 + 2 >= ea.id_limit) a.z = -FLT_MAX;
            if (id0 + 3 >= ea.id_limit) a.w = -FLT_MAX;
          }
          float bv = a.x;
          int bi = id0;
          if (a.y > bv) { bv = a.y; bi = id0 + 1; }
          if (a.z > bv) { bv = a.z; bi = id0 + 2; }
          if (a.w > bv) { bv = a.w; bi = id0 + 3; }
  #pragma unroll
          for (int o = 16; o; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
              bv = ov;
              bi = oi;
            }
          }
          if (lane == 0) ea.amax[static_cast<size_t>(m0 / kBM) * ea.t_stride + n0 + t] = make_float2(bv, __int_as_float(bi));
        }
      }
    } else if (mode == kEpiQkv) {
      const int hd = ea.hd, half = hd >> 1;
      constexpr int pairs = kBM / 2;  // 64 rotation pairs per 128-row tile
      for (int e = threadIdx.x; e < (te - ts) * pairs; e += 128) {
        const int t = ts + e / pairs, p = e % pairs;
        const int hl = p / half, i = p % half;
        const int ra = hl * hd + i, rb = ra + half;
        const int head = (m0 + ra) / hd;
        const float rs = s_rs[t];
        float a = S[t * kBM + ra] * rs, b = S[t * kBM + rb] * rs;
        const int row = n0 + t;
        const int pos = s_pos[t];
        if (head < ea.n_q + ea.n_kv) {
          const float2 cs = ea.rope[static_cast<size_t>(pos) * half + i];
          const float ra2 = a * cs.x - b * cs.y, rb2 = b * cs.x + a * cs.y;
          a = ra2;
          b = rb2;
        }
        if (head < ea.n_q) {
          __nv_bfloat16* qd = ea.q + (static_cast<size_t>(row) * ea.n_q + head) * hd;
          qd[i] = __float2bfloat16_rn(a);
          qd[i + half] = __float2bfloat16_rn(b);
        } else {
          const bool is_v = head >= ea.n_q + ea.n_kv;
          const int kvh = is_v ? head - ea.n_q - ea.n_kv : head - ea.n_q;
          __nv_bfloat16* dst = ea.kv.pool + ea.layer * ea.kv.layer_stride +
                               ((static_cast<size_t>(s_page[t]) * ea.n_kv + kvh) * 2 + (is_v ? 1 : 0)) * kPage * hd +
                               (pos % kPage) * hd;
          dst[i] = __float2bfloat16_rn(a);
          dst[i + half] = __float2bfloat16_rn(b);
        }
      }
    } else {  // kEpiSwiglu: 128-row group = 64 gate rows then 64 up rows
      const int j0 = m0 >> 1;
      for (int e = threadIdx.x; e < (te - ts) * 32; e += 128) {
        const int t = ts + (e >> 5), w = (e & 31) * 2;
        const float rs = s_rs[t];
        const float2 g = *reinterpret_cast<const float2*>(S + t * kBM + w);
        const float2 u = *reinterpret_cast<const float2*>(S + t * kBM + 64 + w);
        const float g0 = g.x * rs, g1 = g.y * rs;
        const float h0 = g0 / (1.f + __expf(-g0)) * (u.x * rs), h1 = g1 / (1.f + __expf(-g1)) * (u.y * rs);
        *reinterpret_cast<__nv_bfloat162*>(ea.h + static_cast<size_t>(n0 + t) * ea.ffn + j0 + w) = __floats2bfloat162_rn(h0, h1);
      }
    }
  if (splits > 1) cluster_wait();  // peers may still be reading this CTA's partial
  __syncthreads();                 // the staging tile is reused by the next weight tile
  }
  if (threadIdx.x == 0) stamp(ea, 5);
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

template <int BN, int ST, int MC = 1>
cudaError_t launch_bn(const GemmOperand& w, const GemmOperand& x, int t, int splits, const EpiArgs& ea,
                      cudaStream_t s) {
  using C = Cfg<BN, ST, MC>;
  static_assert(C::kSmem <= 232448, "shared memory budget");
  static_assert(C::kTmemNeed <= 512, "TMEM budget");
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_kernel<BN, ST, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    cudaFuncSetAttribute(gemm_kernel<BN, ST, MC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  });
  const int kb_total = w.k / kBK;
  const int kps = (kb_total + splits - 1) / splits;
  const int z = (kb_total + kps - 1) / kps;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((w.rows / kBM + MC - 1) / MC, (t + BN - 1) / BN, z);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = z;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = z > 1 ? 2 : 1;  // cluster launch only when the K split needs DSMEM
  // TMA issue layout (FASER_TMA_ISSUE: 0 = one lane, 1 = a lane group per stage (default),
  // 2 = one lane per stage, 3 = one group of lanes splitting every stage's boxes; measured on B200
  // in profiles/r01_tma_issue_ab.txt: 1 is fastest; a warp-uniform variant of 1 (every lane waiting
  // each stage's release in ring order) was slower still and is not kept)
  static const int mode = [] {
    const char* e = std::getenv("FASER_TMA_ISSUE");
    return e ? std::atoi(e) : 1;
  }();
  // activation box rows: one box per stage for row tiles >= 64 (FASER_XBOX=32 keeps 32-row boxes)
  static const int xbox_cap = [] {
    const char* e = std::getenv("FASER_XBOX");
    return e ? std::atoi(e) : 256;
  }();
  int xbox = kXBox;
  const CUtensorMap* xm = &x.map;
  if (x.wide) {
    for (int i = 2; i >= 0; --i) {
      const int r = 64 << i;
      if (((x.wide >> i) & 1) && r <= BN && r <= xbox_cap) {
        xbox = r;
        xm = &x.map_rows[i];
        break;
      }
    }
  }
  const int boxes = MC + BN / xbox;
  const int issue = mode == 0 ? 101 : mode == 2 ? ST * 100 + 1 : mode == 3 ? 100 + (boxes < 32 ? boxes : 32)
                                                                        : ST * 100 + 32 / ST;
  return cudaLaunchKernelEx(&cfg, gemm_kernel<BN, ST, MC>, w.map, *xm, ea, w.rows, kb_total, kps, z, issue, xbox);
}

}  // namespace

namespace {
thread_local bool t_pdl = true;
}
void set_pdl_enabled(bool on) { t_pdl = on; }
bool pdl_enabled() {
  static const bool no_pdl = getenv("FASER_NO_PDL") != nullptr;
  return t_pdl && !no_pdl;
}

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
  cudaError_t e = make_operand(op, x, rows_cap, k, kXBox);
  if (e != cudaSuccess) return e;
  op->wide = 0;
  for (int i = 0; i < 3 && (64 << i) <= rows_cap; ++i) {
    GemmOperand t;
    if ((e = make_operand(&t, x, rows_cap, k, 64 << i)) != cudaSuccess) return e;
    op->map_rows[i] = t.map;
    op->wide |= 1 << i;
  }
  return cudaSuccess;
}

// Launch plan, from a (BN, splits, depth) sweep of graph-timed back-to-back launches on B200
// (tools/gemm_stream.py, profiles/README.md):
//  * enough tiles (>= 120) with one token tile covering all rows: no split, deep pipeline;
//  * otherwise 32-row tiles with a K split of <= 4 (8-CTA clusters schedule badly at 1 CTA/SM),
//    deep pipeline while the grid fits one CTA per SM, 4-stage (2 CTAs/SM) beyond.
constexpr int kMaxSplit = 4;

// Legacy plan (graph-timed sweeps of the MC = 1 kernel; FASER_GEMM_PLAN=legacy).
GemmPlan gemm_plan_legacy(int n_out, int t, int k, int num_sms) {
  GemmPlan p;
  const int mt = n_out / kBM;
  const int kb = k / kBK;
  int cover = 32;
  while (cover < t && cover < 256) cover <<= 1;
  for (int bn = cover; bn >= 64; bn >>= 1) {  // widest token tile that still gives >= 80 tiles
    const int tl = mt * ((t + bn - 1) / bn);
    if (tl >= (bn == cover ? 80 : 120)) {  // a narrower tile re-streams weights per token tile
      p.bn = bn;
      p.splits = 1;
      p.deep = true;
      p.tiles = tl;
      return p;
    }
  }
  if (mt * ((t + 31) / 32) >= 120) {
    p.bn = 32;
    p.splits = 1;
    p.deep = true;
    p.tiles = mt * ((t + 31) / 32);
    return p;
  }
  p.bn = 32;
  const int tiles = mt * ((t + 31) / 32);
  int s = (2 * num_sms) / tiles;
  const int max_s = kb / 4 > 0 ? kb / 4 : 1;  // >= 4 k-blocks (256 of K) per split
  s = s > max_s ? max_s : s;
  s = s > kMaxSplit ? kMaxSplit : s;
  s = s < 1 ? 1 : s;
  const int kps = (kb + s - 1) / s;
  p.splits = (kb + kps - 1) / kps;
  p.tiles = tiles;
  p.deep = tiles * p.splits <= num_sms;
  return p;
}

// Data-driven plan for shapes outside the measured model set: the candidates the kernel set
// instantiates, (bn, mc, depth) x K split, are ranked by their measured slowdown on the two
// nearest shapes of a committed full sweep (plan_table.inc, from profiles/r02_plan_sweep.jsonl:
// 65 shapes of five model families x every plan, 4152 graph-timed launches; distance on
// log2 weight tiles, log2 rows, log2 k-blocks). Leave-one-family-out on that sweep, the pick is
// 1.15x the best plan on average, against 1.26x for the previous fallback (rule classes + legacy
// heuristic) and 1.26-1.32x for fitted analytic cost models. Results are cached
// per (n_out, rows, k).
#include "plan_table.inc"
struct PlanCand {
  int bn, mc;
  bool deep;
};
constexpr PlanCand kPlanCands[] = {{32, 1, true},  {32, 1, false},  {64, 1, true},  {64, 1, false}, {128, 1, true},
                                   {128, 1, false}, {256, 1, true}, {256, 1, false}, {32, 2, true},  {64, 2, true},
                                   {128, 2, true},  {256, 2, true}, {32, 4, true},   {64, 4, true},  {128, 4, true}};

GemmPlan gemm_plan_table(int n_out, int t, int k, double* score) {
  const int mt = n_out / kBM;
  const int kb = k / kBK;
  static std::mutex mu;
  static std::unordered_map<uint64_t, std::pair<GemmPlan, double>> cache;
  const uint64_t key = (static_cast<uint64_t>(n_out) << 40) ^ (static_cast<uint64_t>(t) << 20) ^ static_cast<uint64_t>(k);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      if (score) *score = it->second.second;
      return it->second.first;
    }
  }
  auto feat = [](int n, int rows, int kk, double* f) {
    f[0] = std::log2(n / 128.0);
    f[1] = std::log2(static_cast<double>(rows));
    f[2] = std::log2(kk / 64.0);
  };
  double q[3];
  feat(n_out, t, k, q);
  constexpr int kNear = 2;
  int near[kNear] = {-1, -1};
  double nd[kNear] = {1e30, 1e30};
  const int n_shapes = static_cast<int>(sizeof(kPlanShapes) / sizeof(kPlanShapes[0]));
  for (int i = 0; i < n_shapes; ++i) {
    double f[3];
    feat(kPlanShapes[i][0], kPlanShapes[i][1], kPlanShapes[i][2], f);
    const double d = (f[0] - q[0]) * (f[0] - q[0]) + (f[1] - q[1]) * (f[1] - q[1]) + (f[2] - q[2]) * (f[2] - q[2]);
    for (int j = 0; j < kNear; ++j)
      if (d < nd[j]) {
        for (int m = kNear - 1; m > j; --m) {
          nd[m] = nd[m - 1];
          near[m] = near[m - 1];
        }
        nd[j] = d;
        near[j] = i;
        break;
      }
  }
  static const int kSplitsTry[] = {1, 2, 3, 4, 6, 8};
  constexpr double kMissing = 1098.6;  // log(3) * 1000: a plan the neighbour did not time
  GemmPlan best;
  double best_s = 1e30;
  for (const PlanCand& c : kPlanCands) {
    if (c.mc > 1 && mt < c.mc) continue;
    if (c.bn > 32 && c.bn / 2 >= t) continue;
    for (int sp : kSplitsTry) {
      const int kps = (kb + sp - 1) / sp;
      if (sp > 1 && (kps < 4 || (kb + kps - 1) / kps != sp)) continue;
      double sc = 0.0;
      for (int j = 0; j < kNear; ++j) {
        double e = kMissing;
        if (near[j] >= 0) {
          const int* sh = kPlanShapes[near[j]];
          for (int x = sh[3]; x < sh[3] + sh[4]; ++x) {
            const short* en = kPlanEntries[x];
            if (en[0] == c.bn && en[1] == c.mc && en[2] == (c.deep ? 1 : 0) && en[3] == sp) {
              e = en[4];
              break;
            }
          }
        }
        sc += e;
      }
      sc /= kNear;
      if (sc < best_s) {
        best_s = sc;
        best.bn = c.bn;
        best.mc = c.mc;
        best.deep = c.deep;
        best.splits = sp;
        best.tiles = ((mt + c.mc - 1) / c.mc) * ((t + c.bn - 1) / c.bn);
      }
    }
  }
  {
    std::lock_guard<std::mutex> g(mu);
    cache.emplace(key, std::make_pair(best, best_s / 1000.0));
  }
  if (score) *score = best_s / 1000.0;
  return best;
}

// The models whose GEMM shapes the rule table below was measured on in-stream (configs 3 and 4:
// target and draft projections, LM heads): for them the table (plus the legacy plan it grew from)
// stays in force; every other shape is planned from the measured sweep (gemm_plan_table).
static bool measured_shape(int n_out, int k) {
  static const int kShapes[][2] = {
      {2560, 2048}, {2048, 2048}, {11264, 2048}, {2048, 5632}, {32000, 2048},       // config-3 target
      {2304, 768},  {768, 768},   {6144, 768},   {768, 3072},  {32000, 768},        // config-3 draft
      {6144, 4096}, {4096, 4096}, {28672, 4096}, {4096, 14336}, {128256, 4096},    // config-4 target
      {3072, 2048}, {16384, 2048}, {2048, 8192}, {128256, 2048}};                  // config-4 draft
  for (const auto& sh : kShapes)
    if (sh[0] == n_out && sh[1] == k) return true;
  return false;
}

// Engine plan = the legacy plan plus the shape classes where a graph-timed (bn, mc, split) sweep
// on B200 found a clearly better launch (tools/gemm_sweep.py, profiles/r01_gemm_sweep.jsonl):
//  * wide outputs (LM heads, >= 120 weight tiles) at <= 128 rows: two weight tiles per rows tile
//    (mc = 2), no split: 32000x2048 @128 rows 36.1 -> 29.3 us, 32000x768 @32 13.2 -> 11.4 us;
//  * >= 512 rows and >= 64 tiles: mc = 4 at 128-row token tiles (11264x2048 @512: 52 -> 44 us);
//    (the same-shape sweep's other wins at >= 256 rows did NOT survive in-stream: B=64 verify
//    2.77 -> 3.57 ms, so they are not applied);
//  * <= 32 rows and >= 40 tiles: no K split (6144x768 @32: 10.3 -> 5.7 us);
//  * <= 8 tiles with K >= 3072: 8-way K split (768x3072 @32: 6.7 -> 5.4 us).
// Sharing one rows tile across weight tiles (MC) pays once the rows tile is comparable to a weight
// block: the rows tile is re-read by every weight-tile CTA.
// Experiment hook: FASER_PLAN_OVERRIDE="n_out,k,t_lo,t_hi,bn,mc,splits[,deep];..." forces a plan
// for matching launches (in-stream A/B of plans without rebuilding; deep defaults to 1).
static bool plan_override(int n_out, int t, int k, GemmPlan* p) {
  static const char* env = getenv("FASER_PLAN_OVERRIDE");
  if (!env) return false;
  const char* c = env;
  while (*c) {
    int v[8] = {0, 0, 0, 0, 0, 0, 0, 1}, used = 0, used8 = 0;
    if (sscanf(c, "%d,%d,%d,%d,%d,%d,%d%n", &v[0], &v[1], &v[2], &v[3], &v[4], &v[5], &v[6], &used) != 7) return false;
    if (c[used] == ',' && sscanf(c + used, ",%d%n", &v[7], &used8) == 1) used += used8;
    // only combinations gemm_fused instantiates (and that fit TMEM): otherwise the entry is
    // ignored instead of silently launching a different plan than the one requested
    const bool valid = (v[4] == 32 || v[4] == 64 || v[4] == 128 || v[4] == 256) && (v[5] == 1 || v[5] == 2 || v[5] == 4) &&
                       !(v[4] > 128 && v[5] > 2) && v[4] * v[5] <= 512;
    if (valid && v[0] == n_out && v[1] == k && t >= v[2] && t <= v[3]) {  // invalid entries are ignored
      const int kb = k / kBK, s1 = v[6] < 1 ? 1 : (v[6] > 8 ? 8 : v[6]);
      const int kps = (kb + s1 - 1) / s1;
      p->bn = v[4];
      p->mc = v[5];
      p->splits = (kb + kps - 1) / kps;
      p->deep = v[7] != 0;
      return true;
    }
    c += used;
    while (*c == ';' || *c == ' ') ++c;
  }
  return false;
}

GemmPlan gemm_plan(int n_out, int t, int k, int num_sms) {
  // FASER_GEMM_PLAN: "legacy" = the original heuristic everywhere, "table" = the sweep-driven
  // planner everywhere, unset = rule table for the measured model shapes, sweep-driven otherwise
  static const std::string mode = getenv("FASER_GEMM_PLAN") ? getenv("FASER_GEMM_PLAN") : "";
  const bool legacy = mode == "legacy";
  GemmPlan p = gemm_plan_legacy(n_out, t, k, num_sms);
  if (plan_override(n_out, t, k, &p)) return p;
  if (legacy) return p;
  if (mode == "table" || !measured_shape(n_out, k)) return gemm_plan_table(n_out, t, k, nullptr);
  const int mt = n_out / kBM;
  const int kb = k / kBK;
  int cover = 32;
  while (cover < t && cover < 256) cover <<= 1;
  if (t > 768 && t <= 1024 && k == 2048 && mt >= 64 && mt <= 100) {  // config-3 gate/up at 769..1024 rows
    // 128 x 256 per CTA (with the qkv rule below, profiles/r01_plan_1024_ab.txt)
    p.bn = 256;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (t >= 1024 && mt >= 2 && ((mt + 1) / 2) * ((t + 255) / 256) >= 120) {  // 256 x 256 per CTA (4096 rows: gate/up
    p.bn = 256;                   // 233 -> 183 us = 1.03 PFLOP/s, o 48 -> 34 us, down 101 -> 73 us)
    p.mc = 2;
    p.splits = 1;
    p.deep = true;
  } else if (mt >= 200 && t <= 128) {  // LM heads (and config 4's 28672-row gate/up)
    p.bn = cover;
    p.mc = mt >= 512 ? 4 : 2;            // 128256x2048 @32 rows: mc 4 88.4 vs 95.2 us
    p.splits = 1;
    p.deep = true;
  } else if (t > 64 && t <= 128 && k >= 4096 && n_out >= 4096 && mt <= 32) {
    // config-4 o / down (4096 x 4096, 4096 x 14336) at 128 rows: one 128-row token tile, 4-way K
    // split (in-stream, config 4 B=32: step 12.03 -> 11.29 ms for down alone)
    p.bn = 128;
    p.mc = 1;
    const int kps = (kb + 3) / 4;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 128 && t <= 256 && k >= 4096 && (mt >= 200 || (mt >= 40 && mt <= 64) || (n_out >= 4096 && mt <= 32 && k >= 8192))) {
    // config-4 shapes at 129..256 rows (in-stream, config 4 B=64: step 15.63 -> 14.55 ms):
    // gate/up 128-row tiles x 4 weight tiles, qkv one 128-row tile, down 128 x 2 tiles + 4-way split
    p.bn = 128;
    p.mc = mt >= 200 ? 4 : (mt <= 32 ? 2 : 1);
    const int sp = mt <= 32 ? 4 : 1;
    const int kps = (kb + sp - 1) / sp;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t <= 64 && k >= 8192 && mt <= 16) {  // config-4 draft down (2048 x 8192): 6-way split
    p.bn = t <= 32 ? 32 : 64;
    p.mc = 1;
    const int kps = (kb + 5) / 6;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 32 && t <= 64 && k == 2048 && mt >= 24 && mt <= 32) {  // config-4 draft qkv (3072 x 2048)
    p.bn = 64;
    p.mc = 1;
    const int kps = (kb + 3) / 4;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 64 && t <= 128 && k >= 4096 && k < 8192 && mt <= 16) {  // config-3 down (2048 x 5632)
    // in-stream: verify 1.694 -> 1.681 ms at B = 32 (profiles/r01_plan_down128_ab.txt)
    p.bn = 64;
    p.mc = 1;
    const int kps = (kb + 3) / 4;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 160 && t <= 256 && k >= 4096 && k < 8192 && mt <= 16) {  // config-3 down at 161..256 rows
    // one 128-row token tile, 4-way split (in-stream verify, profiles/r01_plan_256_ab.txt:
    // B = 48 2.63 -> 2.35 ms, B = 56 2.34 -> 2.26 ms, B = 64 2.77 -> 2.59 ms; neutral at 160 rows)
    p.bn = 128;
    p.mc = 1;
    const int kps = (kb + 3) / 4;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 300 && t <= 512 && k >= 4096 && k < 8192 && mt <= 16) {  // config-3 down at 301..512 rows
    // 128-row token tiles, 2-way split (in-stream verify, profiles/r01_plan_512_ab.txt:
    // B = 80 3.92 -> 3.43 ms, B = 96 4.13 -> 3.60 ms, B = 128 4.26 -> 4.20 ms; slower at 288 rows)
    p.bn = 128;
    p.mc = 1;
    const int kps = (kb + 1) / 2;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 448 && t <= 512 && k == 2048 && mt >= 64 && mt <= 100) {  // config-3 gate/up at 449..512 rows
    // 256 x 256 per CTA (B = 128: 4.26 -> 4.09 ms alone; slower at 384 rows)
    p.bn = 256;
    p.mc = 2;
    p.splits = 1;
    p.deep = true;
  } else if (t > 512 && t <= 768 && k >= 2048 && k < 8192 && mt > 8 && mt <= 20 && (mt > 16 || t > 576)) {
    // config-3 qkv / o / down at 513..768 rows: one 128-row token tile per CTA, no split (in-stream
    // verify with the gate/up rule below, profiles/r01_plan_768_ab.txt; o / down keep 64-row tiles
    // up to 576 rows, where 16 x 9 CTAs still fit one wave)
    p.bn = 128;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (t > 512 && t <= 768 && k == 2048 && mt >= 64 && mt <= 100) {  // config-3 gate/up at 513..768 rows
    p.bn = 256;
    p.mc = 2;
    p.splits = 1;
    p.deep = true;
  } else if (t > 768 && t <= 1024 && k == 2048 && mt >= 18 && mt <= 20) {  // config-3 qkv at 769..1024 rows
    // one 128-row token tile per CTA, no split (in-stream verify with the gate/up rule below,
    // profiles/r01_plan_1024_ab.txt: B = 200 6.95 -> 6.20 ms, B = 224 7.78 -> 6.41, B = 256 7.07 -> 6.40);
    // shallow pipeline (2 CTAs/SM) above 960 rows: B = 256 6.40 -> 6.28 ms, but B = 200 (800 rows)
    // 6.21 -> 6.33 ms (profiles/r01_plan_shallow256_ab.txt)
    p.bn = 128;
    p.mc = 1;
    p.splits = 1;
    p.deep = t <= 960;
  } else if (t > 176 && t <= 208 && k == 2048 && mt > 8 && mt <= 16) {  // config-3 o at 177..208 rows
    // 32-row tiles, no split, shallow pipeline (B = 48 2.36 -> 2.24 ms; worse at 160 and 224 rows,
    // profiles/r01_plan_192_ab.txt)
    p.bn = 32;
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 256 && t <= 448 && k == 2048 && ((mt >= 9 && mt <= 20) || (mt >= 64 && mt <= 100))) {
    // config-3 qkv / o / gate/up at 257..448 rows, shallow pipeline (2 CTAs/SM) so the grids that
    // would spill into a second wave at 1 CTA/SM fit one (profiles/r01_plan_448_ab.txt):
    // qkv 64-row tiles, o 32-row tiles, gate/up one 128-row tile (B = 96 3.62 -> ~3.1 ms)
    p.bn = mt >= 64 ? 128 : (mt >= 18 ? 64 : 32);
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 448 && t <= 512 && k == 2048 && mt >= 18 && mt <= 20) {  // config-3 qkv at 449..512 rows
    // 64-row token tiles, shallow pipeline: 160 CTAs at 2 per SM (B = 128 4.04 -> 3.87 ms)
    p.bn = 64;
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 64 && t <= 128 && k == 2048 && mt >= 64 && mt <= 100) {  // config-3 gate/up at 65..128 rows
    // 64-row token tiles with the shallow pipeline: 2 x 88 CTAs at 2 per SM fill the GPU where one
    // 128-row tile per CTA leaves 60 SMs idle (in-stream verify B = 32 1.684 -> 1.651 ms,
    // profiles/r01_plan_gu128_ab.txt)
    p.bn = 64;
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 32 && t <= 64 && k == 768 && mt >= 40 && mt <= 56) {  // config-3 draft gate/up at 33..64 rows
    // 32-row tiles, no split, shallow pipeline (draft B = 64 0.681 -> 0.640 ms, profiles/r01_plan_draft_ab.txt)
    p.bn = 32;
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 96 && t <= 256 && k == 768 && mt >= 40 && mt <= 56) {  // config-3 draft gate/up (6144 x 768)
    // in-stream draft time (profiles/r01_plan_draft_ab.txt): B = 128 0.930 -> 0.892 ms (64-row
    // tiles), B = 256 1.413 -> 1.379 ms (128-row tiles)
    p.bn = t <= 128 ? 64 : 128;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (t > 96 && t <= 128 && k == 3072 && mt <= 8) {  // config-3 draft down (768 x 3072): B = 128 -> 0.910 ms
    p.bn = 64;
    p.mc = 1;
    const int kps = (kb + 3) / 4;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  } else if (t > 240 && t <= 256 && k == 2048 && mt >= 18 && mt <= 20) {  // config-3 qkv at 241..256 rows
    // 32-row token tiles, no split, shallow pipeline (2 CTAs/SM over 160 CTAs): B = 64 2.50 -> 2.41 ms
    // (64-row deep tiles: 2.77 -> 2.67 ms; both worse at 160..224 rows)
    p.bn = 32;
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 224 && t <= 256 && k == 2048 && mt >= 64 && mt <= 100) {  // config-3 gate/up at 225..256 rows
    // one 128-row token tile per CTA, shallow pipeline: 2 x 88 CTAs at 2 per SM (B = 64 2.40 -> 2.37 ms;
    // neutral at 192 / 224 rows, worse at 160)
    p.bn = 128;
    p.mc = 1;
    p.splits = 1;
    p.deep = false;
  } else if (t > 64 && t <= 128 && k >= 4096 && mt >= 40 && mt <= 64) {  // config-4 qkv (6144 x 4096)
    p.bn = 64;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (t >= 512 && mt >= 64) {
    p.bn = 128;
    p.mc = 4;
    p.splits = 1;
    p.deep = true;
  } else if (t <= 32 && mt >= 40 && k <= 1024) {
    p.bn = 32;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (mt <= 8 && k >= 3072 && t <= 128) {
    const int kps = (kb + 7) / 8;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  }
  return p;
}

GemmPlan gemm_plan_prefill(int n_out, int t, int k, int num_sms) {
  // single-prompt prefill (256..1023 rows), from the 576-row sweep (profiles/r01_gemm_sweep_576rows.jsonl)
  static const bool off = getenv("FASER_PREFILL_PLAN") && getenv("FASER_PREFILL_PLAN")[0] == '0';
  GemmPlan p = gemm_plan(n_out, t, k, num_sms);
  // in-stream single-prompt admissions (profiles/r01_prefill_len_ab.txt): the gate/up, qkv and
  // draft-down rules below win at 512..767 rows but lose at 300 / 400 / 1000 rows to the general plan
  if (off || t < 256 || t >= 1024) return p;
  const int mt = n_out / kBM;
  const int kb = k / kBK;
  if (t < 512) {
    // qkv / o / down (2048..2560 outputs) at 256..511 rows: 64-row token tiles keep the grid in one
    // wave (32-row tiles need 16-20 x 10+ CTAs); 300-token admission 4.67 -> 4.01 ms, 400: 4.48 -> 4.36
    if (mt > 8 && mt <= 20 && k >= 2048) {
      p.bn = 64;
      p.mc = 1;
      p.splits = 1;
      p.deep = true;
    }
    return p;
  }
  if (mt <= 16 && mt > 8 && t > 576) {  // o / down (2048 outputs) past 576 rows: 64-row tiles
    // would need 16 x 10+ CTAs = a second wave; one 128-row tile each (600-token admission
    // 5.62 -> 5.26 ms, 700: 6.07 -> 5.47 ms, 760: 6.24 -> 5.60 ms)
    p.bn = 128;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (t >= 768) {
    // general plan
  } else if (mt >= 64 && ((mt + 1) / 2) * ((t + 255) / 256) >= 100) {  // gate/up: 43.9 -> 34.6 us
    p.bn = 256;
    p.mc = 2;
    p.splits = 1;
    p.deep = true;
  } else if (mt >= 18 && k <= 2048) {  // qkv: 23.7 -> 18.6 us, draft qkv 13.5 -> 10.0 us
    p.bn = 128;
    p.mc = 1;
    p.splits = 1;
    p.deep = true;
  } else if (mt <= 8 && k >= 3072) {  // draft down: -> 11.8 us
    p.bn = 128;
    p.mc = 1;
    const int kps = (kb + 3) / 4;
    p.splits = (kb + kps - 1) / kps;
    p.deep = true;
  }
  return p;
}

cudaError_t gemm_fused(const GemmOperand& w, const GemmOperand& x, int t, const GemmPlan& p, const EpiArgs& epi,
                       cudaStream_t s) {
  if (t <= 0) return cudaSuccess;
  if (w.k != x.k) return cudaErrorInvalidValue;
  const bool deep = p.deep;
  if (p.mc == 4) {
    switch (p.bn) {
      case 32: return launch_bn<32, 3, 4>(w, x, t, p.splits, epi, s);
      case 64: return launch_bn<64, 2, 4>(w, x, t, p.splits, epi, s);
      default: return launch_bn<128, 2, 4>(w, x, t, p.splits, epi, s);
    }
  }
  if (p.mc == 2) {
    switch (p.bn) {
      case 32: return launch_bn<32, 5, 2>(w, x, t, p.splits, epi, s);
      case 64: return launch_bn<64, 5, 2>(w, x, t, p.splits, epi, s);
      case 128: return launch_bn<128, 4, 2>(w, x, t, p.splits, epi, s);
      default: return launch_bn<256, 3, 2>(w, x, t, p.splits, epi, s);  // 256 x 256 per CTA (TMEM 512)
    }
  }
  switch (p.bn) {
    case 32: return deep ? launch_bn<32, 8>(w, x, t, p.splits, epi, s) : launch_bn<32, 4>(w, x, t, p.splits, epi, s);
    case 64: return deep ? launch_bn<64, 7>(w, x, t, p.splits, epi, s) : launch_bn<64, 4>(w, x, t, p.splits, epi, s);
    case 128: return deep ? launch_bn<128, 6>(w, x, t, p.splits, epi, s) : launch_bn<128, 3>(w, x, t, p.splits, epi, s);
    default: return deep ? launch_bn<256, 4>(w, x, t, p.splits, epi, s) : launch_bn<256, 2>(w, x, t, p.splits, epi, s);
  }
}

}  // namespace faser

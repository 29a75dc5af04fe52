// llama_attn.cu — K3: varlen causal attention over the paged KV cache.
//
// Each request contributes n_i query rows at consecutive positions pos0_i .. pos0_i+n_i-1
// (1 row per draft step, k_i rows per verify, len-1 rows at prefill). GQA packing: the G
// query heads sharing a KV head are packed with the rows into the MMA M dimension
// (m = row*G + g), so a verify of k_i+... rows x 8 heads is one or a few 16-row tiles and the
// KV page is read once per (request, kv head) tile. QK^T and PV run on mma.sync bf16
// (m16n8k16, fp32 accumulate); K/V pages (64 tokens x head_dim, contiguous) are staged into
// XOR-swizzled shared memory with a 3-stage cp.async pipeline.
// Two work splits:
//   GROUP mode (<= 64 packed rows, decode/verify): one CTA per (request, kv head, 16-row M
//            tile); the 4 warps split each page's four 16-key chunks and merge through smem
//            (short per-warp dependency chains; the extra page reads hit L2).
//   ROWS mode (> 64 packed rows, long verify / prefill): each warp owns a 16-row M tile and
//            walks all keys of the page; CTAs cover 64 packed rows each.
// Few CTAs + long contexts split over KV (flash-decoding); the LAST split CTA to finish a
// (request, kv head, block) merges the partial softmax states in split order (deterministic),
// so there is no separate combine launch.
#include <atomic>
#include <mutex>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "llama.cuh"
#include "sm100.cuh"

namespace faser {
namespace {

constexpr float kNegBig = -1e30f;
constexpr int kMaxPagesPerCta = 256;
// pipeline depth (pages of K+V in flight): latency-bound decode wants many pages in flight
#ifndef FASER_ATTN_STAGES
#define FASER_ATTN_STAGES 3
#endif
template <int HD>
constexpr int kAttnStages = FASER_ATTN_STAGES;

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
// cluster-pair split (GROUP mode): the two halves of a (request, kv head) merge through DSMEM
__device__ __forceinline__ void pair_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sm100::smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_peer(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Swizzled smem tile [64 keys][HD] bf16 in the TMA SWIZZLE_128B box layout: HD/64 boxes of
// [64 rows][128 B]; 16-byte chunk c of row r lives in box c / 8 at chunk (c % 8) ^ (r & 7).
// The cp.async path writes the same layout, so TMA and cp.async pages are interchangeable.
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
  return (chunk >> 3) * (64 * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

// MT = 16-row M tiles per CTA in GROUP mode (128 threads per tile): the tiles of one (request,
// kv head) share every K/V page load instead of re-reading it per tile.
// PPS = pages per pipeline step. PPS = 2 (GROUP mode): each of a tile's 4 warps takes 32
// consecutive keys of a 128-key step, two 16-key chunks under one online-softmax update. That
// halves the rescale / max-reduce / barrier steps per key against PPS = 1 (one 16-key chunk per
// warp per 64-key page).
template <int HD, bool ROWS, int MT = 1, int PPS = 1>
__global__ void __launch_bounds__(128 * MT) attn_kernel(const __grid_constant__ CUtensorMap kvmap, int use_tma,
                                                        RowsDev rows, KvDev kv, int layer, int n_q, int n_kv,
                                                   const __nv_bfloat16* __restrict__ qbuf,
                                                   __nv_bfloat16* __restrict__ obuf, float* __restrict__ part_o,
                                                   float2* __restrict__ part_ml, int* __restrict__ counters,
                                                   int n_split, int rows_cap, int n_blocks, float scale_log2,
                                                   int pair) {
  constexpr int kStages = kAttnStages<HD>;
  constexpr int kChunks = HD / 8;          // 16-byte chunks per K/V row
  constexpr int kTileBytes = 64 * HD * 2;  // one K (or V) page
  constexpr int kStageBytes = PPS * 2 * kTileBytes;
  static_assert(PPS == 1 || (PPS == 2 && !ROWS), "two-page steps are a GROUP-mode layout");
  constexpr int kKS = HD / 16;             // k-steps over head_dim
  constexpr int kDT = HD / 8;              // 8-wide dim tiles of O
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned: the TMA 128-byte swizzle atom (same XOR pattern as swz<64>)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ int s_last;
  __shared__ __align__(8) uint64_t full[kAttnStages<HD>];
  const bool tma = use_tma && PPS == 1;
  // let the next (PDL-launched) GEMM start streaming its weights while attention runs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int req = blockIdx.x, kvh = blockIdx.y;
  const int nr = rows.req_n[req];
  const int gs = 31 - __clz(n_q / n_kv);  // G = n_q / n_kv is a power of two (checked on the host)
  const int gm = (1 << gs) - 1;
  const int G = 1 << gs;
  const int M = nr << gs;
  // pair (cluster of 2 along z, GROUP mode): rank sp walks half of the pages (n_split = 2 page
  // ranges) and rank 0 merges both halves from shared memory (no global partials / counters)
  const int blk = blockIdx.z / n_split, sp = blockIdx.z % n_split;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NT = 128 * MT;  // threads
  const int cta_m0 = ROWS ? blk * 64 : blk * 16 * MT;
  if (cta_m0 >= M) return;
  const int cta_m1 = min(M, cta_m0 + (ROWS ? 64 : 16 * MT));
  // GROUP mode: MT 16-row M tiles per CTA, 4 warps per tile split each page's four 16-key
  // chunks (latency-bound decode: short per-warp dependency chains)
  const int nmt = ROWS ? 4 : 1;
  const int nkg = 4 / nmt;
  const int mt = ROWS ? warp % 4 : warp / 4, kg = ROWS ? 0 : warp % 4;
  const int first = rows.req_first[req], pos0 = rows.req_pos0[req];
  const int slot = rows.req_slot[req];
  const int key_end = pos0 + ((cta_m1 - 1) >> gs) + 1;
  const int tiles = (key_end + 63) / 64;
  const int tps = (tiles + n_split - 1) / n_split;
  const int t0 = sp * tps, t1 = min(tiles, t0 + tps);

  // ---- Q fragments of this warp's 16-row tile
  const int mt0 = cta_m0 + mt * 16;
  const int mlo = mt0 + (lane >> 2), mhi = mlo + 8;
  uint32_t qa[kKS][4];
  {
    const int rlo = mlo >> gs, glo = mlo & gm, rhi = mhi >> gs, ghi = mhi & gm;
    const bool vlo = mlo < cta_m1, vhi = mhi < cta_m1;
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
  const int lim_lo = pos0 + (mlo >> gs), lim_hi = pos0 + (mhi >> gs);  // last visible key per row
  // warp-uniform: last key any row of this warp's tile can see (-1: tile past the live rows)
  const int warp_lim = mt0 < cta_m1 ? pos0 + ((min(mt0 + 15, cta_m1 - 1)) >> gs) : -1;

  float o[kDT][4];
#pragma unroll
  for (int i = 0; i < kDT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_lo = kNegBig, m_hi = kNegBig, l_lo = 0.f, l_hi = 0.f;

  const __nv_bfloat16* kvl = kv.pool + layer * kv.layer_stride;
  // page ids of this CTA's key range, fetched once (a global load per page would sit on the
  // critical path of every pipeline step)
  __shared__ int s_page[kMaxPagesPerCta];
  FASER_DCHECK(t1 <= kv.max_pages, "FASER check: attention req %d slot %d pages %d > %d (pos0 %d rows %d)\n", req,
               slot, t1, kv.max_pages, pos0, nr);
  for (int i = threadIdx.x; i < t1 - t0 && i < kMaxPagesPerCta; i += NT) {
    s_page[i] = kv.ptab[static_cast<int64_t>(slot) * kv.max_pages + t0 + i];
    FASER_DCHECK(static_cast<unsigned>(s_page[i]) < kPageLimit, "FASER check: attention page %d\n", s_page[i]);
  }
  if (tma && threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) sm100::mbar_init(&full[st], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const int64_t layer_rows = kv.layer_stride / HD;
  auto load_tile = [&](int t, int buf, int h) {
    const int page = t - t0 < kMaxPagesPerCta ? s_page[t - t0] : kv.ptab[static_cast<int64_t>(slot) * kv.max_pages + t];
    if (tma) {  // 2 * HD/64 boxes of [64][64] (K and V halves, hardware swizzle), one issuing
                // warp each: a warp's TMA boxes are served one after another (~0.5 us each)
      const int wb = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0 && wb < 2 * (HD / 64)) {
        const int row = static_cast<int>(layer * layer_rows + (static_cast<int64_t>(page) * n_kv + kvh) * 2 * 64);
        if (wb == 0) sm100::mbar_arrive_expect_tx(&full[buf], 2 * kTileBytes);  // the stage's one arrival
        const int kvsel = wb & 1, hb = wb >> 1;  // K / V, 64-column half
        sm100::tma_load_2d(smem + buf * 2 * kTileBytes + kvsel * kTileBytes + hb * 64 * 128, &kvmap, &full[buf],
                           hb * 64, row + kvsel * 64);
      }
      return;
    }
    const uint8_t* gk = reinterpret_cast<const uint8_t*>(kvl + (static_cast<int64_t>(page) * n_kv + kvh) * 2 * 64 * HD);
    const uint8_t* gv = gk + kTileBytes;
    uint8_t* sk = smem + buf * kStageBytes + h * 2 * kTileBytes;
    uint8_t* sv = sk + kTileBytes;
#pragma unroll
    for (int i = threadIdx.x; i < 64 * kChunks; i += NT) {
      const int r = i / kChunks, c = i % kChunks;
      cp_async16(sk + swz<HD>(r, c), gk + i * 16);
      cp_async16(sv + swz<HD>(r, c), gv + i * 16);
    }
  };

  const int nsteps = (t1 - t0 + PPS - 1) / PPS;
  auto load_step = [&](int u) {
#pragma unroll
    for (int h = 0; h < PPS; ++h) {
      const int t = t0 + u * PPS + h;
      if (t < t1) load_tile(t, u % kStages, h);
    }
  };
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < nsteps) load_step(st);
    cp_async_commit();
  }
  for (int u = 0; u < nsteps; ++u) {
    if (tma)
      sm100::mbar_wait(&full[u % kStages], (u / kStages) & 1);
    else
      cp_async_wait<kStages - 2>();
    __syncthreads();  // step u landed for everyone; step u-1's buffer is free
    {
      const int nu = u + kStages - 1;
      if (nu < nsteps) load_step(nu);
      cp_async_commit();
    }
    const uint8_t* stage = smem + (u % kStages) * kStageBytes;
    if constexpr (PPS == 2) {
      // this warp: page h of the step, keys [cb*16, cb*16 + 32) of that page
      const int h = kg >> 1, cb = (kg & 1) * 2;
      const int t = t0 + u * 2 + h;
      const int kbase = t * 64 + cb * 16;
      if (t < t1 && kbase <= warp_lim) {
        const uint8_t* k_s = stage + h * 2 * kTileBytes;
        const uint8_t* v_s = k_s + kTileBytes;
        float s[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
        const int mi = lane >> 3;
#pragma unroll
        for (int kk = 0; kk < kKS; ++kk) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t b[4];
            const int key = (cb + cc) * 16 + 8 * (mi >> 1) + (lane & 7);
            ldsm_x4(b, k_s + swz<HD>(key, kk * 2 + (mi & 1)));
            mma16816(s[2 * cc], qa[kk], b[0], b[1]);
            mma16816(s[2 * cc + 1], qa[kk], b[2], b[3]);
          }
        }
        float mx_lo = kNegBig, mx_hi = kNegBig;
#pragma unroll
        for (int nt2 = 0; nt2 < 4; ++nt2) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int key = kbase + nt2 * 8 + (lane & 3) * 2 + e;
            s[nt2][e] = key <= lim_lo ? s[nt2][e] * scale_log2 : -INFINITY;
            s[nt2][2 + e] = key <= lim_hi ? s[nt2][2 + e] * scale_log2 : -INFINITY;
            mx_lo = fmaxf(mx_lo, s[nt2][e]);
            mx_hi = fmaxf(mx_hi, s[nt2][2 + e]);
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
        uint32_t pa[2][4];
        float sl = 0.f, sh = 0.f;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          float p[2][4];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            p[q][0] = exp2f(s[2 * cc + q][0] - nm_lo);
            p[q][1] = exp2f(s[2 * cc + q][1] - nm_lo);
            p[q][2] = exp2f(s[2 * cc + q][2] - nm_hi);
            p[q][3] = exp2f(s[2 * cc + q][3] - nm_hi);
            sl += p[q][0] + p[q][1];
            sh += p[q][2] + p[q][3];
          }
          pa[cc][0] = pack_bf16(p[0][0], p[0][1]);
          pa[cc][1] = pack_bf16(p[0][2], p[0][3]);
          pa[cc][2] = pack_bf16(p[1][0], p[1][1]);
          pa[cc][3] = pack_bf16(p[1][2], p[1][3]);
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
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
#pragma unroll
          for (int dt = 0; dt < kDT; dt += 2) {
            uint32_t b[4];
            const int key = (cb + cc) * 16 + 8 * (mi & 1) + (lane & 7);
            ldsm_x4_t(b, v_s + swz<HD>(key, dt + (mi >> 1)));
            mma16816(o[dt], pa[cc], b[0], b[1]);
            mma16816(o[dt + 1], pa[cc], b[2], b[3]);
          }
        }
      }
      continue;
    }
    const int t = t0 + u;
    const uint8_t* k_s = stage;
    const uint8_t* v_s = k_s + kTileBytes;
    for (int c = ROWS ? 0 : kg; c < 4; c += (ROWS ? 1 : nkg)) {  // 16-key chunks of the page
      const int kbase = t * 64 + c * 16;
      if (kbase > warp_lim) continue;  // chunk fully past the causal limit of every row of the tile
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
      float mx_lo = kNegBig, mx_hi = kNegBig;
#pragma unroll
      for (int nt2 = 0; nt2 < 2; ++nt2) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = kbase + nt2 * 8 + (lane & 3) * 2 + e;
          s[nt2][e] = key <= lim_lo ? s[nt2][e] * scale_log2 : -INFINITY;
          s[nt2][2 + e] = key <= lim_hi ? s[nt2][2 + e] * scale_log2 : -INFINITY;
          mx_lo = fmaxf(mx_lo, s[nt2][e]);
          mx_hi = fmaxf(mx_hi, s[nt2][2 + e]);
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
      for (int nt2 = 0; nt2 < 2; ++nt2) {
        p[nt2][0] = exp2f(s[nt2][0] - nm_lo);
        p[nt2][1] = exp2f(s[nt2][1] - nm_lo);
        p[nt2][2] = exp2f(s[nt2][2] - nm_hi);
        p[nt2][3] = exp2f(s[nt2][3] - nm_hi);
        sl += p[nt2][0] + p[nt2][1];
        sh += p[nt2][2] + p[nt2][3];
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
  }
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, off);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, off);
  }

  // ---- merge the warps that share an M tile (GROUP mode) through smem: per-row (m, l, O)
  float* so = reinterpret_cast<float*>(smem);  // [4*MT warps][16][HD]
  float* sm = so + 4 * MT * 16 * HD;           // [4*MT][16]
  float* sl_ = sm + 64 * MT;                   // [4*MT][16]
  {
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
      sl_[warp * 16 + rl] = l_lo;
      sl_[warp * 16 + rh] = l_hi;
    }
  }
  __syncthreads();
  // each (packed row, dim) of this CTA: combine its warps -> final (n_split == 1) or partial
  const int ntiles = ROWS ? 4 : MT;
  const int wpt = ROWS ? 1 : nkg;  // warps per tile
  if (!ROWS && pair) {
    pair_sync();  // both halves' per-warp (m, l, O) are in their shared memory
    if (sp == 0) {
      const uint32_t p_so = peer_addr(so, 1), p_sm = peer_addr(sm, 1), p_sl = peer_addr(sl_, 1);
      for (int e = threadIdx.x; e < ntiles * 16 * HD; e += NT) {
        const int tl = e / (16 * HD), r = (e / HD) % 16, col = e % HD;
        const int m = cta_m0 + tl * 16 + r;
        if (m >= cta_m1) continue;
        float mm = kNegBig;
        for (int g = 0; g < wpt; ++g) {
          const int w = tl * 4 + g;
          mm = fmaxf(mm, fmaxf(sm[w * 16 + r], ld_peer(p_sm + 4u * (w * 16 + r))));
        }
        float l = 0.f, acc = 0.f;
        for (int g = 0; g < wpt; ++g) {  // this half's warps, then the peer's (fixed order)
          const int w = tl * 4 + g;
          const float f = exp2f(sm[w * 16 + r] - mm);
          l += sl_[w * 16 + r] * f;
          acc += so[(w * 16 + r) * HD + col] * f;
        }
        for (int g = 0; g < wpt; ++g) {
          const int w = tl * 4 + g;
          const float f = exp2f(ld_peer(p_sm + 4u * (w * 16 + r)) - mm);
          l += ld_peer(p_sl + 4u * (w * 16 + r)) * f;
          acc += ld_peer(p_so + 4u * ((w * 16 + r) * HD + col)) * f;
        }
        const int row = first + (m >> gs), head = kvh * G + (m & gm);
        obuf[(static_cast<int64_t>(row) * n_q + head) * HD + col] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
      }
    }
    pair_sync();  // rank 1's shared memory stays alive until rank 0 has read it
    return;
  }
  for (int e = threadIdx.x; e < ntiles * 16 * HD; e += NT) {
    const int tl = e / (16 * HD), r = (e / HD) % 16, col = e % HD;
    const int m = cta_m0 + tl * 16 + r;
    if (m >= cta_m1) continue;
    float mm = kNegBig;
    for (int g = 0; g < wpt; ++g) mm = fmaxf(mm, sm[(ROWS ? tl : tl * 4 + g) * 16 + r]);
    float l = 0.f, acc = 0.f;
    for (int g = 0; g < wpt; ++g) {
      const int w = ROWS ? tl : tl * 4 + g;
      const float f = exp2f(sm[w * 16 + r] - mm);
      l += sl_[w * 16 + r] * f;
      acc += so[(w * 16 + r) * HD + col] * f;
    }
    const int row = first + (m >> gs), head = kvh * G + (m & gm);
    if (n_split == 1) {
      obuf[(static_cast<int64_t>(row) * n_q + head) * HD + col] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
    } else {
      part_o[((static_cast<int64_t>(sp) * rows_cap + row) * n_q + head) * HD + col] = acc;
      if (col == 0) part_ml[(static_cast<int64_t>(sp) * rows_cap + row) * n_q + head] = make_float2(mm, l);
    }
  }
  if (n_split == 1) return;
  // ---- split-KV: the last CTA of this (request, kv head, block) merges the splits in order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int* cnt = counters + (static_cast<int64_t>(req) * n_kv + kvh) * n_blocks + blk;
    const int prev = atomicAdd(cnt, 1);
    s_last = prev == n_split - 1;
    if (s_last) *cnt = 0;  // self-reset for the next layer / launch
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // per packed row: merged max, and each split's weight exp2(m_s - m) / l  (fixed split order)
  float* sfac = reinterpret_cast<float*>(smem);  // [64 rows][16 splits]
  const int nrow = cta_m1 - cta_m0;
  for (int mr = threadIdx.x; mr < nrow; mr += NT) {
    const int m = cta_m0 + mr;
    const int row = first + (m >> gs), head = kvh * G + (m & gm);
    float2 ml[16];
    float mm = kNegBig;
#pragma unroll
    for (int sp2 = 0; sp2 < 16; ++sp2) {
      if (sp2 < n_split) {
        ml[sp2] = __ldcg(&part_ml[(static_cast<int64_t>(sp2) * rows_cap + row) * n_q + head]);
        mm = fmaxf(mm, ml[sp2].x);
      }
    }
    float l = 0.f;
#pragma unroll
    for (int sp2 = 0; sp2 < 16; ++sp2)
      if (sp2 < n_split) l += ml[sp2].y * exp2f(ml[sp2].x - mm);
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int sp2 = 0; sp2 < 16; ++sp2)
      if (sp2 < n_split) sfac[mr * 16 + sp2] = exp2f(ml[sp2].x - mm) * inv;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nrow * (HD / 4); e += NT) {
    const int mr = e / (HD / 4), c4 = (e % (HD / 4)) * 4;
    const int m = cta_m0 + mr;
    const int row = first + (m >> gs), head = kvh * G + (m & gm);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int sp2 = 0; sp2 < 16; ++sp2) {
      if (sp2 < n_split) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(
            &part_o[((static_cast<int64_t>(sp2) * rows_cap + row) * n_q + head) * HD + c4]));
        const float f = sfac[mr * 16 + sp2];
        acc.x += v.x * f;
        acc.y += v.y * f;
        acc.z += v.z * f;
        acc.w += v.w * f;
      }
    }
    __nv_bfloat16* od = obuf + (static_cast<int64_t>(row) * n_q + head) * HD + c4;
    *reinterpret_cast<__nv_bfloat162*>(od) = __floats2bfloat162_rn(acc.x, acc.y);
    *reinterpret_cast<__nv_bfloat162*>(od + 2) = __floats2bfloat162_rn(acc.z, acc.w);
  }
}

bool want_tma_env() {  // TMA page loads unless FASER_ATTN_TMA=0
  static const bool v = !(getenv("FASER_ATTN_TMA") && getenv("FASER_ATTN_TMA")[0] == '0');
  return v;
}

template <int HD, bool ROWS, int MT = 1, int PPS = 1>
cudaError_t launch(const LlamaShape& m, RowsDev rows, int n_req, int blocks, int n_split, KvDev kv,
                   int layer, const __nv_bfloat16* qbuf, __nv_bfloat16* obuf, float* part_o,
                   float2* part_ml, int* counters, int rows_cap, float scale_log2, cudaStream_t s,
                   int pair = 0) {
  constexpr int kTile = 64 * HD * 2;
  constexpr int kMerge = (4 * MT * 16 * HD + 128 * MT) * 4;
  constexpr int kSmem = (PPS * 2 * kAttnStages<HD> * kTile > kMerge ? PPS * 2 * kAttnStages<HD> * kTile : kMerge) + 1024;
  static std::once_flag attr_once;  // thread-safe: TP ranks launch from several host threads
  std::call_once(attr_once, [] {
    cudaFuncSetAttribute(attn_kernel<HD, ROWS, MT, PPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  });
  dim3 grid(n_req, m.n_kv, blocks * n_split);
  static const CUtensorMap dummy{};  // read-only placeholder when TMA is off
  // TMA page loads (one thread per CTA, hardware swizzle; round 1 measured them equal to the
  // cp.async path): the default whenever the pool has a TMA view (FASER_ATTN_TMA=0: cp.async)
  static const bool want_tma = want_tma_env();
  const bool use_tma = want_tma && kv.tma != nullptr && PPS == 1;
  if (pair) {  // a cluster of two CTAs per (request, kv head, block): n_split = 2 page halves
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_req, m.n_kv, blocks * 2);
    cfg.blockDim = dim3(128 * MT, 1, 1);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 2;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, attn_kernel<HD, ROWS, MT, PPS>, use_tma ? *kv.tma : dummy, use_tma ? 1 : 0, rows,
                              kv, layer, m.n_q, m.n_kv, qbuf, obuf, part_o, part_ml, counters, 2, rows_cap, blocks,
                              scale_log2, 1);
  }
  attn_kernel<HD, ROWS, MT, PPS><<<grid, 128 * MT, kSmem, s>>>(use_tma ? *kv.tma : dummy, use_tma ? 1 : 0, rows, kv, layer,
                                                          m.n_q, m.n_kv, qbuf, obuf, part_o, part_ml, counters,
                                                          n_split, rows_cap, blocks, scale_log2, 0);
  return cudaGetLastError();
}

}  // namespace

cudaError_t lm_attention(const LlamaShape& m, RowsDev rows, int n_req, int max_rows_per_req,
                         int max_ctx, KvDev kv, int layer, const __nv_bfloat16* qbuf,
                         __nv_bfloat16* obuf, float* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (n_req <= 0 || max_rows_per_req <= 0) return cudaSuccess;
  if (m.hd != 64 && m.hd != 128) return cudaErrorInvalidValue;
  const int G = m.n_q / m.n_kv;
  if (G & (G - 1)) return cudaErrorInvalidValue;  // GQA group must be a power of two
  const int Mmax = max_rows_per_req * G;
  const bool rows_mode = Mmax > 64;
  // GROUP mode with > 16 packed rows: two M tiles per CTA (256 threads) share each page load
  static const bool mt1 = getenv("FASER_ATTN_MT1") != nullptr;
  const int mt = (!rows_mode && Mmax > 16 && !mt1) ? 2 : 1;
  const int blocks = rows_mode ? (Mmax + 63) / 64 : (Mmax + 16 * mt - 1) / (16 * mt);
  const int rows_cap = n_req * max_rows_per_req;  // row indices are < sum of req_n <= this
  // scratch = [counters (1 MiB, zeroed at allocation, self-resetting)][part_o][part_ml]
  constexpr size_t kCounterBytes = size_t(1) << 20;
  int* counters = reinterpret_cast<int*>(scratch);
  if (static_cast<size_t>(n_req) * m.n_kv * blocks * 4 > kCounterBytes) return cudaErrorInvalidValue;
  float* body = scratch + kCounterBytes / 4;
  const size_t body_bytes = scratch_bytes - kCounterBytes;
  const int base = n_req * m.n_kv * blocks;
  const int tiles = (max_ctx + 63) / 64;
  int n_split = 1;
  static const int target = getenv("FASER_ATTN_CTAS") ? atoi(getenv("FASER_ATTN_CTAS")) : 148;
  // a split costs a partial write + counter + merge round trip (~4 us with one M tile per CTA,
  // ~7 us with two) against ~0.65 us per page a CTA no longer walks: worth it only for long
  // contexts (profiles/r02_attn_split_small_batch.txt)
  const int min_tiles = mt == 2 ? 24 : 12;
  if (base < target / 2 && tiles >= min_tiles) {
    n_split = (target + base - 1) / base;
    const int max_split = (tiles + 1) / 2 < 16 ? (tiles + 1) / 2 : 16;  // >= 2 pages per split
    if (n_split > max_split) n_split = max_split;
  }
  static std::atomic<int> dbg{getenv("FASER_ATTN_DEBUG") ? atoi(getenv("FASER_ATTN_DEBUG")) : 0};
  if (dbg.load(std::memory_order_relaxed) > 0 && dbg.fetch_sub(1) > 0) {
    fprintf(stderr, "[attn] n_req %d max_rows %d max_ctx %d Mmax %d split %d tma %d group_tc %d rows_tc %d\n", n_req,
            max_rows_per_req, max_ctx, Mmax, n_split, kv.tma != nullptr,
            int(!rows_mode && attn_tc_applies(m, max_rows_per_req, max_ctx, kv)),
            int(rows_mode && attn_tc_rows_applies(m, max_ctx, kv)));
  }
  // tensor-core path (llama_attn_tc.cu) for GQA-packed rows when no KV split is wanted
  if (n_split == 1 && !rows_mode && attn_tc_applies(m, max_rows_per_req, max_ctx, kv))
    return lm_attention_tc(m, rows, n_req, max_rows_per_req, kv, layer, qbuf, obuf, s);
  if (rows_mode && attn_tc_rows_applies(m, max_ctx, kv))
    return lm_attention_tc(m, rows, n_req, max_rows_per_req, kv, layer, qbuf, obuf, s);
  // cluster-pair split for GROUP rows (two CTAs per (request, kv head) walk half the pages each
  // and merge through DSMEM, no global partials) when the doubled grid still leaves every CTA its
  // own SM: two CTAs sharing an SM slow each other's instruction-bound page walk
  // (profiles/r02_attn_pair_split.txt; FASER_ATTN_PAIR = minimum pages, 0 = off)
  static const int pair_min = getenv("FASER_ATTN_PAIR") ? atoi(getenv("FASER_ATTN_PAIR")) : 6;
  const int pair = (!rows_mode && n_split == 1 && pair_min > 0 && tiles >= pair_min && 2 * base <= target) ? 1 : 0;
  const size_t per_split = static_cast<size_t>(rows_cap) * m.n_q * (m.hd * 4 + 8);
  while (n_split > 1 && per_split * n_split > body_bytes) --n_split;
  float* part_o = body;
  float2* part_ml = reinterpret_cast<float2*>(body + static_cast<size_t>(n_split) * rows_cap * m.n_q * m.hd);
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(m.hd));
  if (m.hd == 64) {
    if (rows_mode) return launch<64, true>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s);
    // two-page steps (PPS = 2, FASER_ATTN_WIDE=1)
    static const bool wide = getenv("FASER_ATTN_WIDE") && getenv("FASER_ATTN_WIDE")[0] == '1';
    if (wide && !(want_tma_env() && kv.tma)) {
      if (mt == 2) return launch<64, false, 2, 2>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s, pair);
      return launch<64, false, 1, 2>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s, pair);
    }
    if (mt == 2) return launch<64, false, 2>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s, pair);
    return launch<64, false>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s, pair);
  }
  if (rows_mode) return launch<128, true>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s);
  if (mt == 2) return launch<128, false, 2>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s, pair);
  return launch<128, false>(m, rows, n_req, blocks, n_split, kv, layer, qbuf, obuf, part_o, part_ml, counters, rows_cap, scale_log2, s, pair);
}

}  // namespace faser

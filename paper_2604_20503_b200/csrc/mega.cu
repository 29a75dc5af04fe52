// mega.cu — persistent single-launch forward (see mega.cuh for the phase program).
//
// CTA = 256 threads, one per SM (cooperative launch, ~216 KB shared memory):
//   warp 0 lane 0 : TMA producer. Two cursors over the CTA's job list (one job = one 128x64
//                   weight block of one stream-K unit): the WEIGHT cursor runs ahead across
//                   phases as long as the weight ring has room; the ACTIVATION cursor waits for
//                   the previous phase's grid-wide completion before loading the rows' tile.
//   warp 1 lane 0 : tcgen05.mma issuer (UMMA 128 x N x 16, N = rows rounded to 32), fp32
//                   accumulators double-buffered in TMEM (2 x 256 columns).
//   warp 2        : TMEM allocator.
//   warps 4-7     : epilogue / phase workers: TMEM -> registers, stream-K partial exchange,
//                   fused epilogues (RoPE + KV append, residual + sum of squares, SwiGLU,
//                   LM-head tile argmax), embedding rows, attention units, final argmax.
// Phase completion: every CTA's workers arrive on a per-phase counter after their last write
// of the phase; consumers acquire it before reading. Counters are monotone across launches
// (target = (epoch + 1) * count), so no memset is needed between launches or graph replays.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>
#include <cstdlib>

#include "mega.cuh"
#include "sm100.cuh"
#include "tc_gemm.cuh"

namespace faser {
namespace {

constexpr int kThreads = 256;
constexpr int kEpi0 = 128;                // first worker thread (warps 4..7)
constexpr int kWBytes = 128 * 64 * 2;     // weight block: 128 rows x 64 k (bf16), SWIZZLE_128B
constexpr int kChunk = 32;                // tokens per epilogue staging chunk
constexpr int kArrStride = 32;            // words between phase arrival counters
constexpr int kCntStride = 8;             // words between tile counters
constexpr int kMaxPagesPerUnit = 256;
constexpr float kNegBig = -1e30f;

enum PhaseKind { kPhEmbed = 0, kPhQkv, kPhAttn, kPhO, kPhGu, kPhDown, kPhLm, kPhArgmax };

template <int HD>
struct MCfg {
  static constexpr int kAStages = HD == 64 ? 3 : 2;         // attention K/V page pipeline
  static constexpr int kATile = 64 * HD * 2;                 // one K (or V) page
  static constexpr int kAttBytes = 2 * kAStages * kATile;    // 48 KB (hd 64) / 64 KB (hd 128)
  static constexpr int kRing = HD == 64 ? 160 * 1024 : 144 * 1024;  // weight+rows stage ring
  static constexpr int kOffAtt = kRing;
  static constexpr int kOffMisc = kOffAtt + kAttBytes;
  static constexpr int kMisc = 8192;
  static constexpr int kSmem = 1024 + kOffMisc + kMisc;
  static_assert(kAttBytes >= kChunk * 128 * 4, "epilogue staging aliases the attention region");
};

// ------------------------------------------------------------------ small device helpers
__device__ __forceinline__ void bar_workers() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// debug timeline: CTA `cta` worker event k of phase 4 (trace slots after the per-phase arrays)
#define MEGA_EV(k)                                                                                          \
  do {                                                                                                     \
    if (S.trace && et == 0 && p == 4 && (cta == 0 || cta == 77) && (k) < 32)                               \
      S.trace[static_cast<size_t>(2 * P + 4) * G + 256 + (cta == 0 ? 0 : 32) + (k)] = gtimer();           \
  } while (0)
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Bounded spin: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void spin_until_geq(const unsigned* p, unsigned target) {
  long long n = 0;
  while (static_cast<int>(ld_acquire(p) - target) < 0) {
    if (++n > (1ll << 25)) __trap();
    __nanosleep(n < 8 ? 32 : 128);
  }
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(sm100::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Warp-uniform barrier test / wait: lane 0 tests, the result is broadcast.
__device__ __forceinline__ bool warp_test(uint64_t* bar, uint32_t parity) {
  int ok = (threadIdx.x & 31) == 0 ? (mbar_test(bar, parity) ? 1 : 0) : 0;
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}
__device__ __forceinline__ void warp_wait(uint64_t* bar, uint32_t parity) {
  long long n = 0;
  while (!warp_test(bar, parity)) {
    if (++n > (1ll << 28)) __trap();
  }
}
__device__ __forceinline__ int phase_kind(int p, int L, int* layer) {
  if (p == 0) {
    *layer = 0;
    return kPhEmbed;
  }
  if (p == 1 + 5 * L) {
    *layer = L;
    return kPhLm;
  }
  if (p == 2 + 5 * L) {
    *layer = L;
    return kPhArgmax;
  }
  *layer = (p - 1) / 5;
  return kPhQkv + (p - 1) % 5;
}

// ------------------------------------------------------------------ stream-K partition
// All partition arithmetic is 32-bit (mt * kb * grid < 2^31 for every model here) and the job
// cursor advances incrementally: a 64-bit division per job costs the single issuing thread
// ~1 us and throttles the whole pipeline.
// A job ("super-block") = mc consecutive 128-row weight tiles x one 64-wide k-block, sharing
// one rows tile: the rows are re-read from L2 once per mc weight blocks instead of once per
// block (the per-SM TMA ingest, not HBM, bounds this kernel when the rows tile is as large as
// the weight block).
struct GPhase {
  int mt, kb, wmap, xmap, mode, layer, geff, rot, nb, mc, ng;
};

__device__ __forceinline__ bool gemm_phase(const MegaModelDev& M, int p, int G, int mc, GPhase* g) {
  int l = 0;
  const int k = phase_kind(p, M.layers, &l);
  int n_out = 0, K = 0;
  const int L = M.layers;
  switch (k) {
    case kPhQkv: n_out = (M.n_q + 2 * M.n_kv) * M.hd; K = M.d; g->wmap = 4 * l; g->xmap = 4 * L + 1; g->mode = kEpiQkv; break;
    case kPhO: n_out = M.d; K = M.n_q * M.hd; g->wmap = 4 * l + 1; g->xmap = 4 * L + 9; g->mode = kEpiResid; break;
    case kPhGu: n_out = 2 * M.ffn; K = M.d; g->wmap = 4 * l + 2; g->xmap = 4 * L + 1; g->mode = kEpiSwiglu; break;
    case kPhDown: n_out = M.d; K = M.ffn; g->wmap = 4 * l + 3; g->xmap = 4 * L + 17; g->mode = kEpiResid; break;
    case kPhLm: n_out = M.vocab; K = M.d; g->wmap = 4 * L; g->xmap = 4 * L + 1; g->mode = kEpiLogits; break;
    default: return false;
  }
  g->layer = l;
  g->mt = n_out >> 7;
  g->kb = K >> 6;
  g->mc = mc;
  g->ng = (g->mt + mc - 1) / mc;
  g->nb = g->ng * g->kb;
  int ge = g->nb / M.min_blocks;
  if (ge < 1) ge = 1;
  g->geff = ge < G ? ge : G;
  g->rot = (p * 61) % G;
  return true;
}
__device__ __forceinline__ int vcta(const GPhase& g, int cta, int G) { return (cta - g.rot + G) % G; }
__device__ __forceinline__ int blk_begin(const GPhase& g, int v) {
  return static_cast<int>(static_cast<unsigned>(v) * static_cast<unsigned>(g.nb) / static_cast<unsigned>(g.geff));
}
// virtual CTA owning global super-block b
__device__ __forceinline__ int blk_owner(const GPhase& g, int b) {
  return static_cast<int>((static_cast<unsigned>(b + 1) * static_cast<unsigned>(g.geff) - 1u) / static_cast<unsigned>(g.nb));
}
__device__ __forceinline__ int group_tiles(const GPhase& g, int grp) { return min(g.mc, g.mt - grp * g.mc); }

// Job cursor over this CTA's super-blocks, phase after phase (m = tile group, kk = k-block).
struct JobIt {
  int p, P, cta, G, mc;
  GPhase g;
  int b, b0, b1, m, kk;
  __device__ void seek(const MegaModelDev& M) {
    while (p < P) {
      if (gemm_phase(M, p, G, mc, &g)) {
        const int v = vcta(g, cta, G);
        if (v < g.geff) {
          b0 = b = blk_begin(g, v);
          b1 = blk_begin(g, v + 1);
          if (b < b1) {
            m = b / g.kb;
            kk = b - m * g.kb;
            return;
          }
        }
      }
      ++p;
    }
  }
  __device__ void init(const MegaModelDev& M, int P_, int cta_, int G_, int mc_) {
    p = 0;
    P = P_;
    cta = cta_;
    G = G_;
    mc = mc_;
    seek(M);
  }
  __device__ void next(const MegaModelDev& M) {
    if (++b >= b1) {
      ++p;
      seek(M);
      return;
    }
    if (++kk == g.kb) {
      kk = 0;
      ++m;
    }
  }
  __device__ bool first() const { return b == b0 || kk == 0; }
  __device__ bool last() const { return b == b1 - 1 || kk == g.kb - 1; }
};

// ------------------------------------------------------------------ fused epilogue on a chunk
// Sc = [kChunk tokens][128 tile rows] fp32 (already reduced over the K split); tokens c0..c0+nt.
struct EpiSmem {
  float rs[kMegaMaxT];  // RMSNorm scale of every row (this phase's input residual)
  int pos[kMegaMaxT];
  int page[kMegaMaxT];
};

// Per-phase row prologue, once per phase for all T rows with every load in flight at once:
// RMSNorm scale from the per-128-column sums of squares, and (QKV) position + KV page.
__device__ void phase_prologue(const MegaModelDev& M, const MegaStep& S, int mode, EpiSmem* es, int et) {
  const int T = S.T;
  for (int row = et; row < T; row += 128) {
    if (mode != kEpiResid) {
      const int nch = M.d >> 7;
      float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int c0 = 0; c0 < nch; c0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + u < nch) part[u] += M.ss[static_cast<size_t>(c0 + u) * T + row];
      }
      const float ss = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
      es->rs[row] = rsqrtf(ss / M.d + M.eps);
    }
    if (mode == kEpiQkv) {
      const int pos = S.rows.row_pos[row];
      const int slot = S.rows.req_slot[S.rows.row_req[row]];
      es->pos[row] = pos;
      es->page[row] = M.kv.ptab[static_cast<size_t>(slot) * M.kv.max_pages + pos / kPage];
    }
  }
}

__device__ void epi_chunk(const MegaModelDev& M, const MegaStep& S, const GPhase& g, int m, int c0, int nt,
                          const float* Sc, const EpiSmem* es_, int et) {
  const int T = S.T;
  const int m0 = m * 128;
  const int mode = g.mode;
  struct Shift {  // chunk-relative view of the per-row prologue
    const EpiSmem* e;
    int c0;
    __device__ float rs_(int t) const { return e->rs[c0 + t]; }
    __device__ int pos_(int t) const { return e->pos[c0 + t]; }
    __device__ int page_(int t) const { return e->page[c0 + t]; }
  } es{es_, c0};
  bar_workers();
  const int warp = et >> 5, lane = et & 31;
  const int c4 = lane * 4;
  if (mode == kEpiResid || mode == kEpiLogits) {
    const int n_out = mode == kEpiResid ? M.d : M.vocab;
    for (int t = warp; t < nt; t += 4) {
      const int row = c0 + t;
      float4 a = *reinterpret_cast<const float4*>(Sc + t * 128 + c4);
      if (mode == kEpiResid) {
        const size_t idx = static_cast<size_t>(row) * n_out + m0 + c4;
        const float4 xv = *reinterpret_cast<const float4*>(M.x + idx);
        a = make_float4(xv.x + a.x, xv.y + a.y, xv.z + a.z, xv.w + a.w);
        *reinterpret_cast<float4*>(M.x + idx) = a;
        __nv_bfloat162 b0 = __floats2bfloat162_rn(a.x, a.y), b1 = __floats2bfloat162_rn(a.z, a.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&b0);
        pk.y = *reinterpret_cast<uint32_t*>(&b1);
        *reinterpret_cast<uint2*>(M.xb + idx) = pk;
        float q = (a.x * a.x + a.y * a.y) + (a.z * a.z + a.w * a.w);
#pragma unroll
        for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if (lane == 0) M.ss[static_cast<size_t>(m) * T + row] = q;
      } else {
        const float rs = es.rs_(t);
        a = make_float4(a.x * rs, a.y * rs, a.z * rs, a.w * rs);
        float bv = a.x;
        int bi = m0 + c4;
        if (a.y > bv) { bv = a.y; bi = m0 + c4 + 1; }
        if (a.z > bv) { bv = a.z; bi = m0 + c4 + 2; }
        if (a.w > bv) { bv = a.w; bi = m0 + c4 + 3; }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) {
            bv = ov;
            bi = oi;
          }
        }
        if (lane == 0) M.amax[static_cast<size_t>(m) * T + row] = make_float2(bv, __int_as_float(bi));
      }
    }
  } else if (mode == kEpiQkv) {
    const int hd = M.hd, half = hd >> 1;
    constexpr int pairs = 64;  // rotation pairs per 128-row tile
    for (int e = et; e < nt * pairs; e += 128) {
      const int t = e / pairs, p = e % pairs;
      const int hl = p / half, i = p % half;
      const int ra = hl * hd + i, rb = ra + half;
      const int head = (m0 + ra) / hd;
      const float rs = es.rs_(t);
      float a = Sc[t * 128 + ra] * rs, b = Sc[t * 128 + rb] * rs;
      const int row = c0 + t;
      const int pos = es.pos_(t);
      if (head < M.n_q + M.n_kv) {
        const float2 cs = M.rope[static_cast<size_t>(pos) * half + i];
        const float ra2 = a * cs.x - b * cs.y, rb2 = b * cs.x + a * cs.y;
        a = ra2;
        b = rb2;
      }
      if (head < M.n_q) {
        __nv_bfloat16* qd = M.q + (static_cast<size_t>(row) * M.n_q + head) * hd;
        qd[i] = __float2bfloat16_rn(a);
        qd[i + half] = __float2bfloat16_rn(b);
      } else {
        const bool is_v = head >= M.n_q + M.n_kv;
        const int kvh = is_v ? head - M.n_q - M.n_kv : head - M.n_q;
        __nv_bfloat16* dst = M.kv.pool + g.layer * M.kv.layer_stride +
                             ((static_cast<size_t>(es.page_(t)) * M.n_kv + kvh) * 2 + (is_v ? 1 : 0)) * kPage * hd +
                             (pos % kPage) * hd;
        dst[i] = __float2bfloat16_rn(a);
        dst[i + half] = __float2bfloat16_rn(b);
      }
    }
  } else {  // kEpiSwiglu: 128-row group = 64 gate rows then 64 up rows
    const int j0 = m0 >> 1;
    for (int e = et; e < nt * 32; e += 128) {
      const int t = e >> 5, w = (e & 31) * 2;
      const float rs = es.rs_(t);
      const float2 gg = *reinterpret_cast<const float2*>(Sc + t * 128 + w);
      const float2 u = *reinterpret_cast<const float2*>(Sc + t * 128 + 64 + w);
      const float g0 = gg.x * rs, g1 = gg.y * rs;
      const float h0 = g0 / (1.f + __expf(-g0)) * (u.x * rs), h1 = g1 / (1.f + __expf(-g1)) * (u.y * rs);
      *reinterpret_cast<__nv_bfloat162*>(M.h + static_cast<size_t>(c0 + t) * M.ffn + j0 + w) =
          __floats2bfloat162_rn(h0, h1);
    }
  }
  bar_workers();
}

// ------------------------------------------------------------------ attention unit (K3)
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
template <int HD>
__device__ __forceinline__ int swz(int row, int chunk) {
  return row * (HD * 2) + ((chunk ^ (row & 7)) << 4);
}

// One (request, kv head, block, split) unit of the causal paged attention, executed by the 128
// worker threads (same math and work split as attn_kernel in llama_attn.cu).
template <int HD, bool ROWS, int STAGES>
__device__ void attn_unit(const MegaModelDev& M, const MegaStep& S, int layer, int req, int kvh, int z,
                          uint8_t* smem, int* s_page, int* s_last, int tid) {
  constexpr int kChunks = HD / 8;
  constexpr int kTileBytes = 64 * HD * 2;
  constexpr int kKS = HD / 16;
  constexpr int kDT = HD / 8;
  const RowsDev& rows = S.rows;
  const int n_q = M.n_q, n_kv = M.n_kv, n_split = S.att_split;
  const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(HD));
  bar_workers();  // the previous unit's shared-memory reads are done
  const int nr = rows.req_n[req];
  const int gs = 31 - __clz(n_q / n_kv);
  const int gm = (1 << gs) - 1;
  const int G = 1 << gs;
  const int M_ = nr << gs;
  const int blk = z / n_split, sp = z % n_split;
  const int warp = tid >> 5, lane = tid & 31;
  const int cta_m0 = ROWS ? blk * 64 : blk * 16;
  if (cta_m0 >= M_) return;
  const int cta_m1 = min(M_, cta_m0 + (ROWS ? 64 : 16));
  const int nmt = ROWS ? 4 : 1;
  const int nkg = 4 / nmt;
  const int mt = warp % nmt, kg = warp / nmt;
  const int first = rows.req_first[req], pos0 = rows.req_pos0[req];
  const int slot = rows.req_slot[req];
  const int key_end = pos0 + ((cta_m1 - 1) >> gs) + 1;
  const int tiles = (key_end + 63) / 64;
  const int tps = (tiles + n_split - 1) / n_split;
  const int t0 = sp * tps, t1 = min(tiles, t0 + tps);

  const int mt0 = cta_m0 + mt * 16;
  const int mlo = mt0 + (lane >> 2), mhi = mlo + 8;
  uint32_t qa[kKS][4];
  {
    const int rlo = mlo >> gs, glo = mlo & gm, rhi = mhi >> gs, ghi = mhi & gm;
    const bool vlo = mlo < cta_m1, vhi = mhi < cta_m1;
    const __nv_bfloat16* qlo = M.q + (static_cast<int64_t>(first + (vlo ? rlo : 0)) * n_q + kvh * G + glo) * HD;
    const __nv_bfloat16* qhi = M.q + (static_cast<int64_t>(first + (vhi ? rhi : 0)) * n_q + kvh * G + ghi) * HD;
#pragma unroll
    for (int kk = 0; kk < kKS; ++kk) {
      const int c = kk * 16 + (lane & 3) * 2;
      qa[kk][0] = vlo ? *reinterpret_cast<const uint32_t*>(qlo + c) : 0u;
      qa[kk][1] = vhi ? *reinterpret_cast<const uint32_t*>(qhi + c) : 0u;
      qa[kk][2] = vlo ? *reinterpret_cast<const uint32_t*>(qlo + c + 8) : 0u;
      qa[kk][3] = vhi ? *reinterpret_cast<const uint32_t*>(qhi + c + 8) : 0u;
    }
  }
  const int lim_lo = pos0 + (mlo >> gs), lim_hi = pos0 + (mhi >> gs);
  const int warp_lim = mt0 < cta_m1 ? pos0 + ((min(mt0 + 15, cta_m1 - 1)) >> gs) : -1;

  float o[kDT][4];
#pragma unroll
  for (int i = 0; i < kDT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_lo = kNegBig, m_hi = kNegBig, l_lo = 0.f, l_hi = 0.f;

  const __nv_bfloat16* kvl = M.kv.pool + layer * M.kv.layer_stride;
  for (int i = tid; i < t1 - t0 && i < kMaxPagesPerUnit; i += 128)
    s_page[i] = M.kv.ptab[static_cast<int64_t>(slot) * M.kv.max_pages + t0 + i];
  bar_workers();
  auto load_tile = [&](int t, int buf) {
    const int page = t - t0 < kMaxPagesPerUnit ? s_page[t - t0] : M.kv.ptab[static_cast<int64_t>(slot) * M.kv.max_pages + t];
    const uint8_t* gk = reinterpret_cast<const uint8_t*>(kvl + (static_cast<int64_t>(page) * n_kv + kvh) * 2 * 64 * HD);
    const uint8_t* gv = gk + kTileBytes;
    uint8_t* sk = smem + buf * 2 * kTileBytes;
    uint8_t* sv = sk + kTileBytes;
#pragma unroll
    for (int i = tid; i < 64 * kChunks; i += 128) {
      const int r = i / kChunks, c = i % kChunks;
      cp_async16(sk + swz<HD>(r, c), gk + i * 16);
      cp_async16(sv + swz<HD>(r, c), gv + i * 16);
    }
  };
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (t0 + st < t1) load_tile(t0 + st, st);
    cp_async_commit();
  }
  for (int t = t0; t < t1; ++t) {
    cp_async_wait<STAGES - 2>();
    bar_workers();
    {
      const int nt = t + STAGES - 1;
      if (nt < t1) load_tile(nt, (nt - t0) % STAGES);
      cp_async_commit();
    }
    const uint8_t* k_s = smem + ((t - t0) % STAGES) * 2 * kTileBytes;
    const uint8_t* v_s = k_s + kTileBytes;
    for (int c = ROWS ? 0 : kg; c < 4; c += (ROWS ? 1 : nkg)) {
      const int kbase = t * 64 + c * 16;
      if (kbase > warp_lim) continue;
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
  bar_workers();
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, off);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, off);
  }
  float* so = reinterpret_cast<float*>(smem);  // [4 warps][16][HD]
  float* sm = so + 4 * 16 * HD;                // [4][16]
  float* sl_ = sm + 64;                        // [4][16]
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
  bar_workers();
  const int ntiles = ROWS ? 4 : nmt;
  const int wpt = ROWS ? 1 : nkg;
  const int rows_cap = S.att_rows_cap;
  for (int e = tid; e < ntiles * 16 * HD; e += 128) {
    const int tl = e / (16 * HD), r = (e / HD) % 16, col = e % HD;
    const int m = cta_m0 + tl * 16 + r;
    if (m >= cta_m1) continue;
    float mm = kNegBig;
    for (int g = 0; g < wpt; ++g) mm = fmaxf(mm, sm[(tl + g * nmt) * 16 + r]);
    float l = 0.f, acc = 0.f;
    for (int g = 0; g < wpt; ++g) {
      const int w = tl + g * nmt;
      const float f = exp2f(sm[w * 16 + r] - mm);
      l += sl_[w * 16 + r] * f;
      acc += so[(w * 16 + r) * HD + col] * f;
    }
    const int row = first + (m >> gs), head = kvh * G + (m & gm);
    if (n_split == 1) {
      M.ob[(static_cast<int64_t>(row) * n_q + head) * HD + col] = __float2bfloat16_rn(l > 0.f ? acc / l : 0.f);
    } else {
      S.att_part_o[((static_cast<int64_t>(sp) * rows_cap + row) * n_q + head) * HD + col] = acc;
      if (col == 0) S.att_part_ml[(static_cast<int64_t>(sp) * rows_cap + row) * n_q + head] = make_float2(mm, l);
    }
  }
  if (n_split == 1) return;
  __threadfence();
  bar_workers();
  if (tid == 0) {
    int* cnt = S.att_counters + (static_cast<int64_t>(req) * n_kv + kvh) * S.att_blocks + blk;
    const int prev = atomicAdd(cnt, 1);
    *s_last = prev == n_split - 1;
    if (*s_last) *cnt = 0;
  }
  bar_workers();
  if (!*s_last) return;
  __threadfence();
  float* sfac = reinterpret_cast<float*>(smem);  // [64 rows][16 splits]
  bar_workers();                                 // smem (so/sm) reads above are done
  const int nrow = cta_m1 - cta_m0;
  for (int mr = tid; mr < nrow; mr += 128) {
    const int m = cta_m0 + mr;
    const int row = first + (m >> gs), head = kvh * G + (m & gm);
    float2 ml[16];
    float mm = kNegBig;
#pragma unroll
    for (int sp2 = 0; sp2 < 16; ++sp2) {
      if (sp2 < n_split) {
        ml[sp2] = __ldcg(&S.att_part_ml[(static_cast<int64_t>(sp2) * rows_cap + row) * n_q + head]);
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
  bar_workers();
  for (int e = tid; e < nrow * (HD / 4); e += 128) {
    const int mr = e / (HD / 4), c4 = (e % (HD / 4)) * 4;
    const int m = cta_m0 + mr;
    const int row = first + (m >> gs), head = kvh * G + (m & gm);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int sp2 = 0; sp2 < 16; ++sp2) {
      if (sp2 < n_split) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(
            &S.att_part_o[((static_cast<int64_t>(sp2) * rows_cap + row) * n_q + head) * HD + c4]));
        const float f = sfac[mr * 16 + sp2];
        acc.x += v.x * f;
        acc.y += v.y * f;
        acc.z += v.z * f;
        acc.w += v.w * f;
      }
    }
    __nv_bfloat16* od = M.ob + (static_cast<int64_t>(row) * n_q + head) * HD + c4;
    *reinterpret_cast<__nv_bfloat162*>(od) = __floats2bfloat162_rn(acc.x, acc.y);
    *reinterpret_cast<__nv_bfloat162*>(od + 2) = __floats2bfloat162_rn(acc.z, acc.w);
  }
}

// ------------------------------------------------------------------ the persistent kernel
template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    mega_kernel(const __grid_constant__ MegaModelDev M, const __grid_constant__ MegaStep S) {
  using C = MCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;  // NS stages of [weight block 16 KB | rows tile Tp x 128 B]
  uint8_t* sAtt = smem + C::kOffAtt;
  uint8_t* misc = smem + C::kOffMisc;
  uint64_t* full = reinterpret_cast<uint64_t*>(misc);
  uint64_t* empty = full + 16;
  uint64_t* tfull = empty + 16;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  unsigned* s_epoch = tmem_slot + 1;
  int* s_last = reinterpret_cast<int*>(s_epoch + 1);
  EpiSmem* es = reinterpret_cast<EpiSmem*>(misc + 512);
  int* s_page = reinterpret_cast<int*>(misc + 4096);  // [kMaxPagesPerUnit]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int P = mega_phases(M.layers);
  const int T = S.T;
  const int Tp = (T + 31) & ~31;                 // UMMA N (rows rounded up to the 32-row TMA box)
  const int xbytes = Tp * 128;                   // one activation k-block (Tp rows x 64 bf16)
  const int MC = Tp <= 128 ? 2 : 1;                // weight tiles per rows tile (TMEM: MC*Tp <= 256)
  const int stage_bytes = MC * kWBytes + xbytes;
  const int NS = C::kRing / stage_bytes < 16 ? C::kRing / stage_bytes : 16;
  // phase arrival counters one 128-byte line apart, tile counters 32 bytes apart: pollers of one
  // counter must not queue behind (or hammer) the L2 slice serving another
  unsigned* arrive = M.sync + 32;                       // [P] stride kArrStride
  unsigned* tilecnt = M.sync + 32 + P * kArrStride;     // [P][tile_stride] stride kCntStride

  if (threadIdx.x == 0) {
    for (int s = 0; s < 16; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sm100::mbar_init(&tfull[a], 1);
      sm100::mbar_init(&tempty[a], 1);
    }
    sm100::fence_mbar_init();
    *s_epoch = *reinterpret_cast<volatile unsigned*>(M.sync);
  }
  if (warp == 2) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const unsigned epoch = *s_epoch;
  const unsigned tgt_all = (epoch + 1) * static_cast<unsigned>(G);

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (warp 0)
    // The whole warp runs the loop with warp-uniform control flow (decisions broadcast from
    // lane 0); lane 0 alone issues. A lone spinning lane whose siblings wait at a warp barrier
    // gets time-sliced against them and slows the issue loop several-fold.
    if (lane == 0)
      for (int i = 0; i < 4 * M.layers + 25; ++i) sm100::tma_prefetch(&M.maps[i]);
    const uint64_t pol_w = sm100::policy_evict_first();
    JobIt iw, ix;
    iw.init(M, P, cta, G, MC);
    ix.init(M, P, cta, G, MC);
    uint32_t nw = 0, nx = 0;
    int done = 0;  // phases [0, done) are complete grid-wide
    long long idle = 0;
    while (ix.p < P) {
      bool prog = false;
      // weight cursor: claim the next stage as soon as the MMA released it (any phase ahead)
      if (iw.p < P) {
        const int s = nw % NS;
        if (warp_test(&empty[s], ((nw / NS) & 1) ^ 1)) {
          if (lane == 0) {
            uint8_t* st = ring + s * stage_bytes;
            const int nt = group_tiles(iw.g, iw.m);
            sm100::mbar_arrive_expect_tx(&full[s], nt * kWBytes + xbytes);  // the rows' tile lands later
            for (int i = 0; i < nt; ++i)
              sm100::tma_load_2d_hint(st + i * kWBytes, &M.maps[iw.g.wmap], &full[s], iw.kk * 64,
                                      (iw.m * MC + i) * 128, pol_w);
            if (S.trace && cta == 0 && iw.p == 4 && iw.b - iw.b0 < 32) S.trace[(static_cast<size_t>(2 * P + 4)) * G + (iw.b - iw.b0) * 4 + 0] = gtimer();
          }
          __syncwarp();
          ++nw;
          iw.next(M);
          prog = true;
        }
      }
      // activation cursor: the rows' k-block of a claimed stage, once its phase's inputs exist
      if (nx < nw) {
        if (done < ix.p && !prog) {
          bool adv = false;
          while (done < ix.p) {
            unsigned a = lane == 0 ? ld_acquire(&arrive[done * kArrStride]) : 0u;
            a = __shfl_sync(0xffffffffu, a, 0);
            if (static_cast<int>(a - tgt_all) < 0) break;
            ++done;
            adv = true;
          }
          if (adv && lane == 0) fence_proxy_async_global();
          if (!adv) __nanosleep(64);  // back off: ~148 pollers share this line
          __syncwarp();
        }
        if (done >= ix.p) {
          if (lane == 0) {
            if (S.trace && ix.b == ix.b0) S.trace[(static_cast<size_t>(P) + ix.p) * G + cta] = gtimer();
            // one TMA box of all Tp rows (maps per 32-row multiple): one issue per stage
            uint8_t* st = ring + (nx % NS) * stage_bytes + MC * kWBytes;
            sm100::tma_load_2d(st, &M.maps[ix.g.xmap + (Tp >> 5) - 1], &full[nx % NS], ix.kk * 64, 0);
            if (S.trace && cta == 0 && ix.p == 4 && ix.b - ix.b0 < 32) S.trace[(static_cast<size_t>(2 * P + 4)) * G + (ix.b - ix.b0) * 4 + 1] = gtimer();
          }
          __syncwarp();
          ++nx;
          ix.next(M);
          prog = true;
        }
      }
      if (prog) {
        idle = 0;
      } else if (++idle > (1ll << 28)) {
        __trap();
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (warp 1)
    const uint32_t idesc = sm100::idesc_bf16_f32(128, Tp);
    JobIt it;
    it.init(M, P, cta, G, MC);
    uint32_t n = 0, units = 0;
    while (it.p < P) {
      const bool first = it.first(), last = it.last();
      const uint32_t acc = units & 1;
      if (first) {
        warp_wait(&tempty[acc], ((units >> 1) & 1) ^ 1);
        sm100::tc_fence_after();
      }
      const int s = n % NS;
      warp_wait(&full[s], (n / NS) & 1);
      sm100::tc_fence_after();
      if (lane == 0 && S.trace && cta == 0 && it.p == 4 && it.b - it.b0 < 32) S.trace[(static_cast<size_t>(2 * P + 4)) * G + (it.b - it.b0) * 4 + 2] = gtimer();
      if (lane == 0) {
        const uint64_t db = sm100::desc_sw128(sm100::smem_u32(ring + s * stage_bytes + MC * kWBytes));
        const int nt = group_tiles(it.g, it.m);
        for (int i = 0; i < nt; ++i) {
          const uint64_t da = sm100::desc_sw128(sm100::smem_u32(ring + s * stage_bytes + i * kWBytes));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            sm100::mma_bf16(tmem + acc * 256 + i * Tp, da + 2 * k, db + 2 * k, idesc, (!first || k > 0) ? 1u : 0u);
        }
        sm100::mma_commit(&empty[s]);  // one commit per stage: releases weight + rows tile together
        if (last) sm100::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (last) ++units;
      ++n;
      it.next(M);
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- workers
    const int et = threadIdx.x - kEpi0;
    const int ew = et >> 5;
    float* Sc = reinterpret_cast<float*>(sAtt);  // [kChunk][128] staging (aliases attention smem)
    uint32_t units = 0;
    for (int p = 0; p < P; ++p) {
      if (p > 0) {
        if (et == 0) {
          spin_until_geq(&arrive[(p - 1) * kArrStride], tgt_all);
          __threadfence();
        }
        bar_workers();
      }
      int layer = 0;
      const int kind = phase_kind(p, M.layers, &layer);
      GPhase g;
      if (kind == kPhEmbed) {
        const int nch = M.d / 128;
        const int items = T * nch;
        for (int i = cta * 4 + ew; i < items; i += 4 * G) {
          const int r = i / nch, c = i % nch;
          const int col = c * 128 + lane * 4;
          const uint2 e = *reinterpret_cast<const uint2*>(M.emb + static_cast<size_t>(S.rows.row_tok[r]) * M.d + col);
          const __nv_bfloat162 e0 = *reinterpret_cast<const __nv_bfloat162*>(&e.x);
          const __nv_bfloat162 e1 = *reinterpret_cast<const __nv_bfloat162*>(&e.y);
          const float4 v = make_float4(__low2float(e0), __high2float(e0), __low2float(e1), __high2float(e1));
          *reinterpret_cast<float4*>(M.x + static_cast<size_t>(r) * M.d + col) = v;
          *reinterpret_cast<uint2*>(M.xb + static_cast<size_t>(r) * M.d + col) = e;
          float q = (v.x * v.x + v.y * v.y) + (v.z * v.z + v.w * v.w);
#pragma unroll
          for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
          if (lane == 0) M.ss[static_cast<size_t>(c) * T + r] = q;
        }
      } else if (kind == kPhArgmax) {
        const int nt = M.vocab / 128;
        for (int r = cta * 4 + ew; r < T; r += 4 * G) {
          float bv = -FLT_MAX;
          int bi = 0x7fffffff;
          for (int m = lane; m < nt; m += 32) {
            const float2 pv = __ldcg(&M.amax[static_cast<size_t>(m) * T + r]);
            const int pi = __float_as_int(pv.y);
            if (pv.x > bv || (pv.x == bv && pi < bi)) {
              bv = pv.x;
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
          if (lane == 0) S.argmax_out[r] = bi;
        }
      } else if (kind == kPhAttn) {
        const int per_req = S.att_blocks * S.att_split;
        const int nu = S.n_req * M.n_kv * per_req;
        const int rot = (p * 61) % G;
        for (int u = (cta - rot + G) % G; u < nu; u += G) {
          const int req = u / (M.n_kv * per_req), rem = u % (M.n_kv * per_req);
          const int kvh = rem / per_req, z = rem % per_req;
          if (S.att_rows_mode)
            attn_unit<HD, true, C::kAStages>(M, S, layer, req, kvh, z, sAtt, s_page, s_last, et);
          else
            attn_unit<HD, false, C::kAStages>(M, S, layer, req, kvh, z, sAtt, s_page, s_last, et);
        }
        bar_workers();
      } else if (gemm_phase(M, p, G, MC, &g)) {
        const int v = vcta(g, cta, G);
        if (v < g.geff) {
          MEGA_EV(0);
          phase_prologue(M, S, g.mode, es, et);
          bar_workers();
          MEGA_EV(1);
          int nev = 2;
          const int b0 = blk_begin(g, v), b1 = blk_begin(g, v + 1);
          float* ws = M.ws + static_cast<size_t>(p & 1) * M.ws_slots * (128 * kMegaMaxT);
          const int Tq = (T + 3) & ~3;                           // partial row stride (float4 aligned)
          const size_t tstride = static_cast<size_t>(128) * Tq;  // one partial tile [128 rows][Tq]
          // pass 1: drain every unit's accumulators (TMEM) in MMA order; a group owned by one
          // CTA is finished right away, a split group publishes its partial tiles and signals
          // each tile's counter. No waiting on other CTAs here, so contributions never queue
          // behind a reduction.
          for (int b = b0; b < b1;) {
            const int grp = b / g.kb;
            const int grp_end = (grp + 1) * g.kb;
            const int vf = blk_owner(g, grp * g.kb);
            const int nc = blk_owner(g, grp_end - 1) - vf + 1;
            const int ntile = group_tiles(g, grp);
            const uint32_t acc = units & 1;
            // one polling thread with back-off (128 threads spinning on the mbarrier would steal
            // the barrier unit from the producer / TMA completions of the mainloop)
            if (et == 0) {
              long long spins = 0;
              while (!mbar_test(&tfull[acc], (units >> 1) & 1)) {
                __nanosleep(64);
                if (++spins > (1ll << 26)) __trap();
              }
            }
            bar_workers();
            MEGA_EV(nev); ++nev;
            sm100::tc_fence_after();
            for (int i = 0; i < ntile; ++i) {
              const int m = grp * g.mc + i;
              const uint32_t tbase = tmem + acc * 256 + i * Tp + (static_cast<uint32_t>(ew * 32) << 16);
              if (nc == 1) {
                for (int c0 = 0; c0 < T; c0 += kChunk) {
                  float va[16], vb[16];
                  sm100::tmem_ld16(tbase + c0, va);
                  sm100::tmem_ld16(tbase + c0 + 16, vb);
#pragma unroll
                  for (int q = 0; q < 16; ++q) {
                    Sc[q * 128 + et] = va[q];
                    Sc[(16 + q) * 128 + et] = vb[q];
                  }
                  bar_workers();
                  epi_chunk(M, S, g, m, c0, min(kChunk, T - c0), Sc, es, et);
                }
              } else {
                // partial tile row-major [row][Tq]: this thread's row, 16 tokens per TMEM load
                float* mine = ws + (static_cast<size_t>(v + grp) * g.mc + i) * tstride + static_cast<size_t>(et) * Tq;
                for (int c0 = 0; c0 < Tq; c0 += 16) {
                  float va[16];
                  sm100::tmem_ld16(tbase + c0, va);
#pragma unroll
                  for (int q = 0; q < 16; q += 4)
                    if (c0 + q < Tq) __stcg(reinterpret_cast<float4*>(mine + c0 + q), make_float4(va[q], va[q + 1], va[q + 2], va[q + 3]));
                }
              }
            }
            sm100::tc_fence_before();
            if (nc > 1) __threadfence();
            bar_workers();
            if (et == 0) {
              sm100::mbar_arrive(&tempty[acc]);
              if (nc > 1)
                for (int i = 0; i < ntile; ++i)
                  atomicAdd(&tilecnt[(static_cast<size_t>(p) * M.tile_stride + grp * g.mc + i) * kCntStride], 1u);
            }
            ++units;
            MEGA_EV(nev); ++nev;
            b = grp_end < b1 ? grp_end : b1;
          }
          MEGA_EV(20);
          // pass 2: each contributor of a split group reduces (fixed contributor order) and
          // finishes its 4-aligned slice of the tokens once every contributor has published.
          for (int b = b0; b < b1;) {
            const int grp = b / g.kb;
            const int grp_end = (grp + 1) * g.kb;
            b = grp_end < b1 ? grp_end : b1;
            const int vf = blk_owner(g, grp * g.kb);
            const int nc = blk_owner(g, grp_end - 1) - vf + 1, j = v - vf;
            if (nc == 1) continue;
            const int ts = ((j * T / nc) >> 2) << 2;
            const int te = j == nc - 1 ? T : (((j + 1) * T / nc) >> 2) << 2;
            if (ts >= te) continue;
            const int ntile = group_tiles(g, grp);
            if (et == 0) {
              for (int i = 0; i < ntile; ++i)
                spin_until_geq(&tilecnt[(static_cast<size_t>(p) * M.tile_stride + grp * g.mc + i) * kCntStride],
                               (epoch + 1) * static_cast<unsigned>(nc));
              __threadfence();
            }
            bar_workers();
            MEGA_EV(nev); ++nev;
            // slot of contributor jj for tile i: ((vf + jj + grp) * mc + i); thread = tile row
            const size_t jstride = static_cast<size_t>(g.mc) * tstride;
            for (int i = 0; i < ntile; ++i) {
              const int m = grp * g.mc + i;
              const float* rowp = ws + (static_cast<size_t>(vf + grp) * g.mc + i) * tstride + static_cast<size_t>(et) * Tq;
              for (int c0 = ts; c0 < te; c0 += kChunk) {
                const int ntk = min(kChunk, te - c0);
                float4 acc4[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) acc4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int j0 = 0; j0 < nc; j0 += 2) {  // two contributors' loads in flight at once
                  float4 va[8], vb[8];
                  const bool two = j0 + 1 < nc;
#pragma unroll
                  for (int q = 0; q < 8; ++q) {
                    va[q] = 4 * q < ntk ? __ldcg(reinterpret_cast<const float4*>(rowp + j0 * jstride + c0 + 4 * q)) : make_float4(0.f, 0.f, 0.f, 0.f);
                    vb[q] = (two && 4 * q < ntk) ? __ldcg(reinterpret_cast<const float4*>(rowp + (j0 + 1) * jstride + c0 + 4 * q)) : make_float4(0.f, 0.f, 0.f, 0.f);
                  }
#pragma unroll
                  for (int q = 0; q < 8; ++q) {  // contributor order j0, j0+1 (deterministic)
                    acc4[q].x += va[q].x; acc4[q].y += va[q].y; acc4[q].z += va[q].z; acc4[q].w += va[q].w;
                    if (two) { acc4[q].x += vb[q].x; acc4[q].y += vb[q].y; acc4[q].z += vb[q].z; acc4[q].w += vb[q].w; }
                  }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  if (4 * q < ntk) {
                    Sc[(4 * q) * 128 + et] = acc4[q].x;
                    Sc[(4 * q + 1) * 128 + et] = acc4[q].y;
                    Sc[(4 * q + 2) * 128 + et] = acc4[q].z;
                    Sc[(4 * q + 3) * 128 + et] = acc4[q].w;
                  }
                }
                bar_workers();
                epi_chunk(M, S, g, m, c0, ntk, Sc, es, et);
              }
            }
          }
        }
      }
      MEGA_EV(30);
      // phase done: make this CTA's writes visible (generic and async proxy), then arrive
      fence_proxy_async_global();
      __threadfence();
      bar_workers();
      if (et == 0) {
        if (S.trace) S.trace[static_cast<size_t>(p) * G + cta] = gtimer();
        atomicAdd(&arrive[p * kArrStride], 1u);
      }
    }
  }
  __syncwarp();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&M.sync[1], 1u);
    if (prev == tgt_all - 1) atomicExch(&M.sync[0], epoch + 1);
  }
}

template <int HD>
cudaError_t launch_mega(const MegaModelDev& m, const MegaStep& st, int grid, cudaStream_t s) {
  using C = MCfg<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mega_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr_[1];
  attr_[0].id = cudaLaunchAttributeCooperative;
  attr_[0].val.cooperative = 1;
  cfg.attrs = attr_;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mega_kernel<HD>, m, st);
}

}  // namespace

cudaError_t mega_attn_plan(const LlamaShape& m, int n_req, int max_rows, int max_ctx, float* scratch,
                           size_t scratch_bytes, MegaStep* st) {
  // identical work split to lm_attention (llama_attn.cu)
  const int G = m.n_q / m.n_kv;
  const int Mmax = max_rows * G;
  const bool rows_mode = Mmax > 64;
  const int blocks = rows_mode ? (Mmax + 63) / 64 : (Mmax + 15) / 16;
  const int rows_cap = n_req * max_rows;
  constexpr size_t kCounterBytes = size_t(1) << 20;
  if (static_cast<size_t>(n_req) * m.n_kv * blocks * 4 > kCounterBytes) return cudaErrorInvalidValue;
  float* body = scratch + kCounterBytes / 4;
  const size_t body_bytes = scratch_bytes - kCounterBytes;
  const int base = n_req * m.n_kv * blocks;
  const int tiles = (max_ctx + 63) / 64;
  int n_split = 1;
  static const int target = getenv("FASER_ATTN_CTAS") ? atoi(getenv("FASER_ATTN_CTAS")) : 148;
  if (base < target / 2 && tiles >= 4) {
    n_split = (target + base - 1) / base;
    const int max_split = (tiles + 1) / 2 < 16 ? (tiles + 1) / 2 : 16;
    if (n_split > max_split) n_split = max_split;
  }
  const size_t per_split = static_cast<size_t>(rows_cap) * m.n_q * (m.hd * 4 + 8);
  while (n_split > 1 && per_split * n_split > body_bytes) --n_split;
  st->att_rows_mode = rows_mode ? 1 : 0;
  st->att_blocks = blocks;
  st->att_split = n_split;
  st->att_rows_cap = rows_cap;
  st->att_counters = reinterpret_cast<int*>(scratch);
  st->att_part_o = body;
  st->att_part_ml = reinterpret_cast<float2*>(body + static_cast<size_t>(n_split) * rows_cap * m.n_q * m.hd);
  return cudaSuccess;
}

cudaError_t mega_forward(const MegaModelDev& m, const MegaStep& st, int grid, cudaStream_t s) {
  if (st.T < 1 || st.T > kMegaMaxT) return cudaErrorInvalidValue;
  if (m.hd == 64) return launch_mega<64>(m, st, grid, s);
  if (m.hd == 128) return launch_mega<128>(m, st, grid, s);
  return cudaErrorInvalidValue;
}

}  // namespace faser

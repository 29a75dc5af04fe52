// mega.cuh — persistent single-launch forward of a Llama-style model (draft step or verify).
//
// One cooperative launch (one CTA per SM) runs the whole forward as a sequence of phases:
//   embed | per layer: qkv (+RoPE, paged KV append) | attention | o (+residual) |
//   gate/up (+SwiGLU) | down (+residual) | LM head (+per-tile argmax) | argmax reduce
// separated by grid-wide phase arrivals. Projection phases are swap-AB tcgen05 GEMMs whose
// (m-tile, k-block) weight blocks are split evenly over the CTAs (stream-K); the TMA producer
// streams weight blocks of LATER phases into a shared-memory ring while the current phase is
// still finishing (weights never depend on activations), so the HBM weight stream does not stop
// at phase boundaries the way it does between separate kernel launches. Partial tiles of a
// stream-K split are reduced deterministically (fixed contributor order) by the contributors
// themselves, each on a slice of the tokens. The k-partition depends only on (matrix, SM count),
// never on the number of rows, so a row's result does not depend on which other rows are in
// the batch (batch-invariant, as the early-exit design requires).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "llama.cuh"

namespace faser {

constexpr int kMegaMaxT = 256;  // rows per mega forward (one UMMA N tile, double-buffered TMEM)

// Static per (model, work buffers); lives in kernel parameter space.
struct MegaModelDev {
  const CUtensorMap* maps;  // [4*layers + 25]: per layer {qkv, o, gu, down}, lm, then the xb / ob / h
                            // row tiles with boxes of 32, 64, ..., 256 rows (8 maps each)
  const __nv_bfloat16* emb;
  const float2* rope;
  KvDev kv;
  int d, layers, n_q, n_kv, hd, ffn, vocab;
  float eps;
  float* x;
  __nv_bfloat16* xb;
  float* ss;  // [d/128][T]
  __nv_bfloat16* q;
  __nv_bfloat16* ob;
  __nv_bfloat16* h;
  float2* amax;         // [vocab/128][T]
  float* ws;            // stream-K partials: 2 parities x ws_slots x (128 x kMegaMaxT) fp32
  int ws_slots;
  unsigned* sync;       // [0] epoch, [1] exit count, [32..) phase arrivals (128 B apart), tile counters (32 B apart)
  int tile_stride;      // counters per phase
  int min_blocks;       // minimum super-blocks per stream-K unit (bounds the partial-tile traffic)
};

// Per launch.
struct MegaStep {
  RowsDev rows;
  int T, n_req, max_rows, max_ctx;
  int* argmax_out;
  // attention plan (same work split as lm_attention)
  int att_rows_mode, att_blocks, att_split, att_rows_cap;
  float* att_part_o;
  float2* att_part_ml;
  int* att_counters;
  unsigned long long* trace;  // optional (FASER_MEGA_TRACE): [2][P][grid] phase-end / first-rows-load globaltimer
};

// Number of phases and sync words for a model with `layers` layers.
__host__ __device__ inline int mega_phases(int layers) { return 3 + 5 * layers; }
inline size_t mega_sync_words(int layers, int tile_stride) {
  return 32 + static_cast<size_t>(mega_phases(layers)) * (32 + 8 * static_cast<size_t>(tile_stride));
}
// Partial-workspace floats needed for `grid` CTAs and at most `max_mt` m-tiles per phase.
inline int mega_ws_slots(int grid, int max_mt) { return 2 * grid + max_mt; }
inline size_t mega_ws_floats(int grid, int max_mt) {
  return 2ull * static_cast<size_t>(mega_ws_slots(grid, max_mt)) * 128 * kMegaMaxT;
}

cudaError_t mega_attn_plan(const LlamaShape& m, int n_req, int max_rows, int max_ctx, float* scratch,
                           size_t scratch_bytes, MegaStep* st);
cudaError_t mega_forward(const MegaModelDev& m, const MegaStep& st, int grid, cudaStream_t s);

}  // namespace faser

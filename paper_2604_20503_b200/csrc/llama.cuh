// llama.cuh — device layout + launchers for the Llama-style draft/target pair (configs 3-5).
//
// The reference has no transformer: its "draft/target pair" is LayeredToyLM.
// For configs 3-5 the build supplies random-init bf16 Llama-shaped models whose weights are a
// pure function of (seed, tensor tag, element index) so that the CPU fp32 oracle
// (oracle/llama_oracle.c) regenerates exactly the same bf16 values. Acceptance is made
// tunable by a "bigram" construction (the analogue of the toy's eta, toylm.cpp:76-85): the
// embedding of token t is bigram_scale * W_lm[g(t)] + noise, with g(t) = (a*t + b) mod V
// shared by both models, so both models lean towards g(x) and agree when the layer stack does
// not override it.
//
// HBM layout (per engine):
//   weights   : per model, one bf16 arena; per layer [wqkv | wo | wgu | wd] row-major
//               (K-major for the swap-AB GEMM). wgu interleaves gate/up in 64-row groups.
//   KV pages  : per model, [layer][page][kv_head][K|V][P=64][head_dim] bf16; a request's
//               page table maps position -> page (shared across layers).
//   rows      : ragged batch of the current forward (slot, position, token per row) +
//               per-request (first row, n rows); n_rows lives in device memory so early-exit
//               compaction can shrink it without a host round trip.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "faser/engine.h"

namespace faser {

constexpr int kPage = 64;  // tokens per KV page

// Cheap device-side range checks on data-dependent indices (token ids, page ids): a violation
// prints the site and traps (a kernel error on the host) instead of corrupting memory.
#define FASER_DCHECK(cond, ...)  \
  do {                           \
    if (!(cond)) {               \
      printf(__VA_ARGS__);       \
      __trap();                  \
    }                            \
  } while (0)
constexpr unsigned kTokLimit = 1u << 20;   // > every vocabulary here
constexpr unsigned kPageLimit = 1u << 24;

struct LlamaShape {
  int d, layers, n_q, n_kv, hd, ffn, vocab;
  float rope_theta, eps;
  float bigram_scale, embed_noise, init_std;
  double hard_fraction;
  uint64_t seed;
  int qkv_out() const { return (n_q + 2 * n_kv) * hd; }
};

// Element generator shared with the oracle: Irwin-Hall(4) on 16-bit lanes of a SplitMix64
// hash, scaled and rounded to bf16 (exact IEEE ops only, so CPU and GPU agree bit-for-bit).
__host__ __device__ inline uint64_t lm_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Tensor tags (per model, per layer): tag = kind * 4096 + layer.
enum : uint32_t { kTagLm = 1, kTagEmbNoise = 2, kTagQkv = 3, kTagO = 4, kTagGate = 5, kTagUp = 6, kTagDown = 7, kTagHard = 8 };

struct LayerW {
  const __nv_bfloat16* wqkv;  // [qkv_out][d]
  const __nv_bfloat16* wo;    // [d][n_q*hd]
  const __nv_bfloat16* wgu;   // [2*ffn][d], 64-row groups: gate j0..j0+63, up j0..j0+63, ...
  const __nv_bfloat16* wd;    // [d][ffn]
};

// Ragged batch of one forward pass (device arrays; capacity rows_cap / req_cap).
struct RowsDev {
  int* n_rows;     // [1] live rows (shrinks under early-exit compaction)
  int* row_req;    // [rows] request index within this forward
  int* row_pos;    // [rows] absolute position of the row's input token
  int* row_tok;    // [rows] input token id
  int* row_j;      // [rows] index of the row within its request (drafted position)
  int* req_first;  // [reqs] first row (compacted order)
  int* req_n;      // [reqs] rows of the request
  int* req_slot;   // [reqs] engine slot (page table row)
  int* req_pos0;   // [reqs] position of the request's first row
};

struct KvDev {
  __nv_bfloat16* pool;  // [layers][pages][n_kv][2][kPage][hd]
  const int* ptab;      // [slots][max_pages]
  int max_pages;
  int64_t layer_stride;  // elements per layer
  // TMA view of the pool as [rows = layers*pages*n_kv*2*64][hd] with 64x64 boxes and the 128 B
  // swizzle the attention kernel's shared-memory layout uses (hd 128: two boxes per page row
  // block; nullptr = cp.async)
  const CUtensorMap* tma = nullptr;
};

// ------------------------------------------------------------------ launchers
// elements [offset, offset + n) of the tensor (offset: a TP row shard)
cudaError_t lm_init_matrix(__nv_bfloat16* w, int64_t n, uint64_t seed, uint32_t tag, float std,
                           cudaStream_t s, int64_t offset = 0);
// columns [c0, c0 + kl) of a row-major [rows][k_full] tensor (row-parallel TP shard)
cudaError_t lm_init_cols(__nv_bfloat16* w, int64_t rows, int64_t k_full, int64_t c0, int64_t kl, uint64_t seed,
                         uint32_t tag, float std, cudaStream_t s);
// wgu in the interleaved order (gate rows tagged kTagGate, up rows kTagUp, both [ffn][d]); `ffn`
// local rows starting at global FFN row f0 (TP column shard).
cudaError_t lm_init_gate_up(__nv_bfloat16* wgu, int ffn, int d, uint64_t seed, uint32_t tag_layer,
                            float std, cudaStream_t s, int64_t f0 = 0);
// emb[t] = bf16(bigram_scale * lm[g(t)] + noise(t))
cudaError_t lm_init_embedding(__nv_bfloat16* emb, const __nv_bfloat16* lm, const LlamaShape& m,
                              uint32_t ga, uint32_t gb, cudaStream_t s);

// x[r] = emb[row_tok[r]] (fp32 residual), xb = bf16 copy (the GEMM operand; RMSNorm is folded
// into the consuming GEMM's epilogue), ss[c][r] = sum of squares of 128-column chunk c.
cudaError_t lm_embed(const LlamaShape& m, const __nv_bfloat16* emb, RowsDev rows, int rows_cap,
                     float* x, __nv_bfloat16* xb, float* ss, cudaStream_t s);
// argmax_lowest over the per-128-vocab-tile (max, lowest id) partials of the logits epilogue.
cudaError_t lm_argmax_reduce(int n_tiles, RowsDev rows, int rows_cap, const float2* amax, int* out,
                             cudaStream_t s);
// GQA-packed verify / decode rows on tcgen05 (llama_attn_tc.cu): one CTA per (request, kv head),
// S and O in TMEM; used by lm_attention when G >= 4, <= 64 packed rows, no KV split.
bool attn_tc_applies(const LlamaShape& m, int max_rows_per_req, int max_ctx, const KvDev& kv);
// prefill / long-row blocks on the same kernel in 128-row tiles (ROWS work of lm_attention)
bool attn_tc_rows_applies(const LlamaShape& m, int max_ctx, const KvDev& kv);
cudaError_t lm_attention_tc(const LlamaShape& m, RowsDev rows, int n_req, int max_rows_per_req, KvDev kv, int layer,
                            const __nv_bfloat16* qbuf, __nv_bfloat16* obuf, cudaStream_t s);
// Causal attention of every row over its request's paged KV (GQA packed, mma.sync bf16).
cudaError_t lm_attention(const LlamaShape& m, RowsDev rows, int n_req, int max_rows_per_req,
                         int max_ctx, KvDev kv, int layer, const __nv_bfloat16* qbuf,
                         __nv_bfloat16* obuf, float* scratch, size_t scratch_bytes, cudaStream_t s);

}  // namespace faser

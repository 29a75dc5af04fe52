// tc_gemm.cuh — host interface of the tcgen05 swap-AB GEMM with fused epilogues (tc_gemm.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "llama.cuh"

namespace faser {

// A bf16 row-major [rows][k] matrix with its TMA descriptor (SWIZZLE_128B, box 64 x box_rows).
struct GemmOperand {
  CUtensorMap map;
  // activation operands: the same tensor with 64 / 128 / 256-row boxes (map has 32-row boxes).
  // One box per pipeline stage for wide row tiles: a TMA box costs ~0.5 us of issue latency per
  // issuing warp regardless of its size (tools/tma_probe.cu, profiles/r02_tma_box_probe.jsonl),
  // so four 32-row boxes per stage cap a CTA at a quarter of the 128-row box's ingest.
  CUtensorMap map_rows[3];
  int wide = 0;  // bit i: map_rows[i] (64 << i rows per box) valid (box rows <= tensor rows)
  const void* base = nullptr;
  int rows = 0;
  int k = 0;
};

cudaError_t make_weight_operand(GemmOperand* op, const void* w, int n_out, int k);  // box 128 rows
cudaError_t make_act_operand(GemmOperand* op, const void* x, int rows_cap, int k);  // box 32 rows
cudaError_t make_operand(GemmOperand* op, const void* base, int rows, int k, int box_rows);

enum EpiMode : int {
  kEpiStore = 0,   // out[t][n] = acc * rs[t]                        (fp32)
  kEpiResid = 1,   // x[t][n] += acc; xb = bf16(x); ss_out[mtile][t] = sum_n x^2 over the tile
  kEpiQkv = 2,     // RoPE(q,k) at row_pos; q -> bf16 [t][n_q*hd]; k,v -> paged KV cache
  kEpiSwiglu = 3,  // h[t][j] = bf16(silu(gate*rs) * up*rs), gate/up interleaved in 64-row groups
  kEpiLogits = 4,  // logits[t][v] = acc*rs (fp32) + per-tile (max, lowest idx) per token
  kEpiRank = 5,    // fused exit-test estimator: per (vocab tile, token) count of ids outranking the
                   // token's drafted id d (z_v > z_d, or = and v < d), z_d from zd_src; no logits
};

// Everything the fused epilogue may need (unused fields ignored per mode).
struct EpiArgs {
  int mode = kEpiStore;
  int t_stride = 0;          // row capacity of this launch (host T)
  const int* n_rows = nullptr;  // live rows (device), nullptr -> t_stride
  // RMSNorm folded into the epilogue: acc *= rsqrt(sum_c ss_in[c][t] / d_norm + eps)
  const float* ss_in = nullptr;
  int ss_chunks = 0, d_norm = 0;
  float eps = 0.f;
  float* out = nullptr;                  // kEpiStore
  __nv_bfloat16* out_bf16 = nullptr;     // kEpiStore: bf16 output instead of `out` (TP partials)
  float* x = nullptr;                    // kEpiResid
  __nv_bfloat16* xb = nullptr;           // kEpiResid
  float* ss_out = nullptr;               // kEpiResid [n_out/128][t_stride]
  RowsDev rows{};                        // kEpiQkv
  const float2* rope = nullptr;          // kEpiQkv [pos][hd/2] (cos, sin)
  KvDev kv{};                            // kEpiQkv
  int layer = 0, n_q = 0, n_kv = 0, hd = 0;
  __nv_bfloat16* q = nullptr;            // kEpiQkv [t][n_q*hd]
  __nv_bfloat16* h = nullptr;            // kEpiSwiglu [t][ffn]
  int ffn = 0;
  float* logits = nullptr;               // kEpiLogits [t][n_out]; nullptr: argmax partials only
  float2* amax = nullptr;                // kEpiLogits [n_out/128][t_stride] (value, idx bits)
  int id_off = 0;                        // kEpiLogits: id of output row 0 (vocab-parallel shard)
  int id_limit = 0;                      // kEpiLogits: ids >= id_limit are padding (0 = none)
  // kEpiRank: z_d of token t = zd_src[t * 128 + t % 128] (a [t][128] block-diagonal GEMM over the
  // gathered rows W[d_t], same accumulation order as this LM head), d_t = row_d[t] (-1: no test);
  // counts -> rank_cnt[n_out/128][t_stride]. logits (optional) are written as in kEpiLogits.
  const float* zd_src = nullptr;
  const int* row_d = nullptr;
  int* rank_cnt = nullptr;
  // kEpiLogits sampling (faser_set_sampling): inv_tau > 0 perturbs the argmax operand of token t
  // (row n0 + t) to logit * inv_tau + Gumbel(sample_key(samp_seed, req_ids[rows.row_req[row]],
  // rows.row_pos[row] + 1), id): the per-tile (max, id) partials then hold a sample of
  // softmax(logits / tau) (Gumbel-max); the logits written stay the raw ones. rows must be set.
  const int64_t* req_ids = nullptr;
  unsigned long long samp_seed = 0;
  float inv_tau = 0.f;
  int t_begin = 0;                       // first token of this launch (token tiles start here)
  int w_after_wait = 0;                  // 1: the weights are written by the previous kernel (no
                                         // weight prefetch before griddepcontrol.wait)
  // optional timeline (tools/layer_chain.py): per CTA 8 globaltimer stamps [cta][8] = entry, after
  // griddepcontrol.wait, first stage landed, accumulators complete, split-K reduced, exit
  unsigned long long* trace = nullptr;
};

// Launch plan: token-tile width and K split (the splits of a tile form one thread-block cluster
// and reduce through DSMEM). Fixed per forward so surviving rows' numerics do not depend on
// early-exit pruning.
struct GemmPlan {
  int bn = 32;
  int splits = 1;
  int tiles = 0;
  bool deep = true;  // deep pipeline (~200 KB smem, 1 CTA / SM) vs 4-stage (2 CTAs / SM)
  int mc = 1;        // 128-row weight tiles per CTA sharing one rows tile (1, 2, 4)
};
GemmPlan gemm_plan(int n_out, int t, int k, int num_sms);
// Sweep-driven plan (tc_gemm.cu, plan_table.inc); score (optional) = the pick's mean log slowdown
// on its nearest measured shapes.
GemmPlan gemm_plan_table(int n_out, int t, int k, double* score);
// Plan for a prefill forward (one or a few prompts, 128..8192 rows, no logits): 128-row token
// tiles from 256 rows up (the same-shape sweep's winners, which did not survive in the verify
// stream but are measured here on prefill separately).
GemmPlan gemm_plan_prefill(int n_out, int t, int k, int num_sms);

// Programmatic dependent launch for this host thread's subsequent launches (GEMMs and the fused
// draft control kernels); on by default, FASER_NO_PDL=1 disables it process-wide.
void set_pdl_enabled(bool on);
bool pdl_enabled();

// D[n][t] = sum_k W[n][k] X[t][k] over T = min(*n_rows, t) rows, epilogue per `epi`.
// Launched with programmatic stream serialization: the prologue overlaps the previous kernel;
// all dependent reads happen after griddepcontrol.wait.
cudaError_t gemm_fused(const GemmOperand& w, const GemmOperand& x, int t, const GemmPlan& p,
                       const EpiArgs& epi, cudaStream_t s);

}  // namespace faser

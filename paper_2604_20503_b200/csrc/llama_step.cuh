// llama_step.cuh — per-step device state of the Llama-style serving path and the launchers of
// the small control kernels around the forwards (draft row prep, verify row prep, K4 early-exit
// rank-count + frontier compaction, K5 fused greedy accept + commit + rollback).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "faser/engine.h"
#include "llama.cuh"

namespace faser {

// Per-slot request state (SoA, HBM), the Llama analogue of SlotState.
struct LmSlots {
  int32_t* tok;      // [slots][max_seq] prompt ++ committed
  int32_t* len;      // [slots] context length (prompt + committed)
  int32_t* ncomm;    // [slots]
  int32_t* max_out;  // [slots]
  int32_t* done;     // [slots]
  int32_t* exempt;   // [slots] exempt_position (-1 unset)
  int32_t max_seq;
};

// Per-request (this step, sorted by k' descending) early-exit / draft state.
struct LmReqState {
  int32_t* slot;        // [n] engine slot
  int32_t* k;           // [n] k_i' = min(k_i, remaining)
  int32_t* spec;        // [n] controller's k_i (reported)
  int32_t* live_idx;    // [n] position in the live (batch) order for results
  int64_t* req_id;      // [n]
  int32_t* drafted;     // [n][FASER_MAX_SPEC]
  int32_t* count;       // [n] drafted length (EOS stop)
  int32_t* active;      // [n] early-exit frontier
  int32_t* gate_layers; // [n]
  int32_t* n_pl;        // [n]
  int32_t* pl;          // [n][FASER_MAX_SPEC] prune layers (VerifyOutcome::prune_layers)
  int32_t* prune_layer; // [n][FASER_MAX_SPEC] layer at which row j was pruned (L if never)
  int32_t* pr;          // [n][2] last pruned_at (j, layer), -1 if none
  uint32_t* failmask;   // [n] exit-test failures at the current gated layer
  int32_t* truth;       // [rows] final argmax per verify row (compacted order)
  int32_t* truth_rj;    // [n][FASER_MAX_SPEC] final argmax by (request, drafted position)
  int32_t* span;        // [n] chunked verify: drafted positions covered by the chunks the request
                        // was verified in (its frontier's reach)
};

// Frontier-chunked (FULL) verify state shared by the two lanes of one step (device ints):
//   alive        requests still on the frontier after the latest verified chunk (verify lane
//                writes, the draft lane reads it to cancel chunks nobody will verify)
//   rec[2q]      requests on the frontier with rows in chunk q, rec[2q+1] its rows;
//                rec[2*nchunks] requests whose every drafted token was verified and accepted
//   resets[q]    requests whose frontier chunk q's verification reset (rejection or prune)
//   step_dec[t]  draft step t: 0 undecided, 1 run, 2 cancelled (reset observed before it started)
struct LaneState {
  int32_t* alive;
  int32_t* rec;
  int32_t* step_dec;
  int32_t* resets;
};

struct StepCtl {
  int n;           // requests this step
  int layers;      // target layers (L)
  int eos;
  int early_exit;  // 1: verify_with_early_exit semantics
  int exempt_rule; // 1: exempt = committed_before + pruned_at.first for the next round;
                   // 2: recovery on prune (beyond the reference: the first pruned row runs to
                   //    full depth and its argmax is committed, no exemption)
};

// draft step t: rows = sorted requests [0, n_t); row r = request r, 1 row each at position
// len_r - 1 + t, input token = last committed (t == 0) or drafted[r][t-1].
cudaError_t lm_draft_prep(LmSlots sl, LmReqState rq, RowsDev rows, int n_t, int t, cudaStream_t s);
// fused draft step control (one warp per row, PDL launches): step 0's rows + embeddings; and
// after step t: argmax over the LM head's per-tile partials -> drafted[r][t], then step t+1's
// rows + embeddings for the first n_next rows (argmax_reduce + draft_post + draft_prep + embed).
cudaError_t lm_draft_begin(LmSlots sl, LmReqState rq, RowsDev rows, int n_t, const __nv_bfloat16* emb, int d,
                           float* x, __nv_bfloat16* xb, float* ss, cudaStream_t s);
// With `lane` (overlapped mode), step t+1 is cancelled when no request is left on the frontier
// (lane.alive == 0) at the time step t finishes: its rows are emptied so the forward's kernels exit
// at once (the reference's draft cancellation after a reset, overlap.cpp:58-62).
cudaError_t lm_draft_advance(LmSlots sl, LmReqState rq, RowsDev rows, const float2* amax, int n_tiles, int n_t,
                             int t, int n_next, const __nv_bfloat16* emb, int d, float* x, __nv_bfloat16* xb,
                             float* ss, cudaStream_t s, const LaneState* lane = nullptr);
// verify rows' tokens + embeddings (verify_tokens + embed fused; one warp per row)
cudaError_t lm_verify_begin(LmSlots sl, LmReqState rq, RowsDev rows, int rows_cap, const __nv_bfloat16* emb, int d,
                            float* x, __nv_bfloat16* xb, float* ss, cudaStream_t s);
// final per-row argmax of the verify LM head -> truth[row] and truth_rj[req][j] (fused scatter)
cudaError_t lm_verify_argmax(RowsDev rows, int n_tiles, int rows_cap, const float2* amax, int* truth, int* truth_rj,
                             cudaStream_t s);
// after draft step t: drafted[r][t] = argmax[r].
cudaError_t lm_draft_post(LmReqState rq, const int* argmax, int n_t, int t, cudaStream_t s);
// verify rows (whole verify or one overlap chunk): row tokens from ctx.back() / drafted.
cudaError_t lm_verify_tokens(LmSlots sl, LmReqState rq, RowsDev rows, int rows_cap, cudaStream_t s);
// once all tokens are drafted: drafted lengths (EOS stop) and the early-exit state.
cudaError_t lm_verify_init(LmReqState rq, int n, int layers, int eos, cudaStream_t s);
// final argmax rows -> truth_rj[request][j].
cudaError_t lm_truth_scatter(RowsDev rows, const int* argmax, int* truth_rj, int rows_cap, cudaStream_t s);
// K4 fused estimator (no T x V logits): rank_prep writes each live row's drafted id (row_d, -1
// off the frontier) and gathers W_lm[d] into wg [rows][d]; a block-diagonal GEMM over wg gives z_d;
// the LM head's kEpiRank epilogue counts, per 128-id tile, the ids outranking d; exit_rank sums
// the tiles and sets the failmask bit when the count reaches k_thr.
cudaError_t lm_rank_prep(LmReqState rq, RowsDev rows, const __nv_bfloat16* wlm, int d, __nv_bfloat16* wg,
                         int* row_d, int rows_cap, cudaStream_t s);
cudaError_t lm_exit_rank(LmSlots sl, LmReqState rq, RowsDev rows, const int* cnt, int n_tiles, int t_stride,
                         int k_thr, int rows_cap, cudaStream_t s);
// K4 frontier: per request earliest failing row prunes the suffix; compacts the row set.
// src_of[new_row] = old row; the residual (x fp32, xb bf16, ss per-chunk sums of squares) is
// gathered through scratch buffers of the same shapes.
// q0 = first drafted position of the rows (0, or the chunk start in the overlapped mode).
// recover = 1 (exempt_rule 2): the first pruned row stays to full depth (recovery token).
cudaError_t lm_frontier_compact(LmSlots sl, LmReqState rq, RowsDev rows, int n, int layer,
                                int* src_of, cudaStream_t s, int q0 = 0, int recover = 0, int layers = 0);
// Overlapped (FULL) verify, before chunk q (drafted positions [q0, q0 + rows)): a request stays on
// the frontier iff no earlier row was pruned (active > q0), rejected (drafted != truth) or EOS;
// otherwise its rows of the chunk are cancelled (reset, overlap.cpp:44-91). The chunk's rows are
// compacted in place; lane.alive / lane.rec[2q..2q+1] record the frontier. first = 1 for chunk 0
// also initialises the per-request early-exit state (active = k).
cudaError_t lm_chunk_frontier(LmReqState rq, RowsDev rows, int n, int q, int q0, int first, int layers, int eos,
                              LaneState lane, cudaStream_t s);
// After the last chunk: drafted length (EOS stop over the drafted tokens, as the serial path),
// active = min(active, count), survivors and per-chunk resets (chunk = frontier chunk size).
cudaError_t lm_chunk_finalize(LmReqState rq, int n, int eos, int nchunks, int chunk, LaneState lane, cudaStream_t s);
cudaError_t lm_gather_rows(RowsDev rows, const int* src_of, int d, int t_stride, float* x,
                           __nv_bfloat16* xb, float* ss, float* xs, __nv_bfloat16* xbs, float* sss,
                           cudaStream_t s);
// K5: greedy acceptance (+ early-exit outcome bookkeeping) + commit + exempt rule.
cudaError_t lm_accept_commit(LmSlots sl, LmReqState rq, RowsDev rows, StepCtl ctl,
                             faser_round_result* results, cudaStream_t s);
// page-table scatter: ptab[slot*max_pages + idx] = page for each (slot, idx, page) triple.
cudaError_t lm_ptab_scatter(int* ptab, int max_pages, const int* triples, int n, cudaStream_t s);
// admission: copy prompts into the slot rows and initialise slot state.
struct LmAdmit {
  const int32_t* src;
  int32_t slot, len, max_out, reserved;
};
cudaError_t lm_admit(LmSlots sl, const LmAdmit* admits, int n, cudaStream_t s);
// prefill rows: tokens of the prompt prefix (positions 0..len-2) read from the slot rows.
cudaError_t lm_prefill_tokens(LmSlots sl, RowsDev rows, int rows_cap, cudaStream_t s);

}  // namespace faser

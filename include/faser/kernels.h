/*
 * faser/kernels.h — kernel-level C ABI of the B200 data path (device pointers, caller's
 * stream). The serving engine (engine.h) drives the same launchers; these entry points
 * exist so each kernel can be checked against its oracle and timed in isolation.
 * All pointers are device pointers; `stream` is a cudaStream_t (NULL = legacy stream).
 * Status codes as in engine.h; a missing GPU is FASER_ECUDA (never a CPU fallback).
 */
#ifndef FASER_KERNELS_H
#define FASER_KERNELS_H

#include <stdint.h>

#include "faser/engine.h"

#ifdef __cplusplus
extern "C" {
#endif

/* out[t][n] = sum_k w[n][k] * x[t][k]; w bf16 [n_out][k], x bf16 [t][k], out fp32 [t][n_out].
 * tcgen05 swap-AB GEMM (verify K2 / draft K1 projections). splits = 0 picks the engine's
 * split-K heuristic. n_out % 128 == 0, k % 64 == 0. */
faser_status faser_k_gemm_bf16(const void* w, const void* x, float* out, int32_t n_out,
                               int32_t t, int32_t k, int32_t splits, void* stream);

/* Same with an explicit launch plan: bn in {32, 64, 128, 256} rows per tile (0 = auto),
 * + 1000 * depth (1 shallow, 2 deep) + 10000 * mc (weight tiles per CTA sharing a rows tile:
 * 1, 2, 4), and splits in [1, 8] (0 = auto). For plan sweeps / microbenchmarks. */
faser_status faser_k_gemm_bf16_plan(const void* w, const void* x, float* out, int32_t n_out,
                                    int32_t t, int32_t k, int32_t bn, int32_t splits, void* stream);
/* The launch plan the engine uses for an [n_out x k] weight and t rows: out = {bn, splits, mc,
 * deep}. Host-only (no device needed). */
faser_status faser_k_gemm_plan(int32_t n_out, int32_t t, int32_t k, int32_t* out4);
/* The sweep-driven planner's plan for the same shape (out4 as above; score = the pick's mean log
 * slowdown on its two nearest measured shapes), whatever FASER_GEMM_PLAN selects for the engine
 * (tc_gemm.cu gemm_plan_table; CPU-callable). */
faser_status faser_k_gemm_plan_table(int32_t n_out, int32_t t, int32_t k, int32_t* out4, double* score);
/* faser_k_gemm_bf16_plan with a per-CTA timeline: trace[cta][8] globaltimer stamps (entry, after
 * griddepcontrol.wait, first stage landed, accumulators complete, split-K reduced, exit); the
 * grid is (weight tiles / mc, row tiles, splits), cta = (z * gy + y) * gx + x. */
faser_status faser_k_gemm_bf16_trace(const void* w, const void* x, float* out, int32_t n_out, int32_t t,
                                     int32_t k, int32_t bn, int32_t splits, void* stream,
                                     unsigned long long* trace);

/* K3: causal attention of n_req ragged query blocks over the paged KV cache (one layer).
 * q bf16 [rows][n_q][hd]; kv bf16 pool [pages][n_kv][2 (K,V)][64][hd]; ptab int32
 * [n_req][max_pages] (request i uses ptab row i); request i has req_n[i] query rows starting at
 * row req_first[i], at positions req_pos0[i] .. req_pos0[i]+req_n[i]-1, attending to keys
 * [0, pos]. out bf16 [rows][n_q][hd]. scratch: device workspace (>= 2 MiB, first MiB zeroed
 * before the first call). n_q / n_kv must be a power of two, hd in {64, 128}. */
faser_status faser_k_attention(const void* q, const void* kv, const int32_t* ptab, int32_t max_pages,
                               int32_t n_req, const int32_t* req_first, const int32_t* req_n,
                               const int32_t* req_pos0, int32_t max_rows, int32_t max_ctx,
                               int32_t n_q, int32_t n_kv, int32_t hd, void* out, void* scratch,
                               int64_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FASER_KERNELS_H */

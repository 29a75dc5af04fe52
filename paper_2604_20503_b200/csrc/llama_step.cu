// llama_step.cu — control kernels of the Llama-style serving step.
//
//   draft prep/post      : SpeculativeEngine::draft_tokens (sdcore.cpp:45-59) as a ragged loop:
//                          step t runs the requests whose budget min(k_i, remaining) > t.
//   verify prep          : verify row i,j has input token ctx.back() (j = 0) or drafted[j-1]
//                          and predicts drafted[j] (full_verify, sdcore.cpp:61-81).
//   exit test (K4)       : token_exit_test (exitctl.cpp:56-68) on the LM head of the
//                          intermediate residual: prune iff >= K(layer) ids outrank drafted[j]
//                          (ties: lower id outranks). No Top-K and no T x V logits: rank_prep
//                          gathers W_lm[d], a block-diagonal GEMM gives z_d in the LM head's own
//                          accumulation order, the LM head's epilogue counts outranking ids per
//                          128-id tile (tc_gemm.cu kEpiRank) and exit_rank sums the tiles.
//   frontier (K4)        : verify_with_early_exit's per-layer scan (sdcore.cpp:111-132):
//                          earliest failing j prunes rows j.. of that request; surviving rows are
//                          compacted so the remaining layers' GEMM/attention tiles shrink.
//   accept + commit (K5) : survivors exact (sdcore.cpp:134-148), force-verify of token 0
//                          (:150-166), full_layers_run (:168-169), commit (:182-197), and the
//                          exempt-position rule; KV "rollback" is the new context length (pages
//                          past it are released by the host).
#include <cuda_runtime.h>

#include <cstdint>

#include "llama_step.cuh"
#include "tc_gemm.cuh"

namespace faser {
namespace {

constexpr int kMS = FASER_MAX_SPEC;

__global__ void draft_prep_kernel(LmSlots sl, LmReqState rq, RowsDev rows, int n_t, int t) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) *rows.n_rows = n_t;
  if (r >= n_t) return;
  const int slot = rq.slot[r];
  const int base = sl.len[slot] - 1;
  const int pos = base + t;
  rows.row_req[r] = r;
  rows.row_pos[r] = pos;
  rows.row_j[r] = t;
  rows.req_first[r] = r;
  rows.req_n[r] = 1;
  rows.req_slot[r] = slot;
  rows.req_pos0[r] = pos;
  rows.row_tok[r] = t == 0 ? sl.tok[static_cast<int64_t>(slot) * sl.max_seq + base]
                           : rq.drafted[r * kMS + t - 1];
}

// Embedding of one row by one warp: x = emb[tok] (fp32), xb = bf16 copy, ss[c][r] = sum of
// squares of 128-column chunk c (the next GEMM folds RMSNorm from it).
__device__ __forceinline__ void embed_row_warp(const __nv_bfloat16* __restrict__ emb, int tok, int r, int d,
                                               int t_stride, float* __restrict__ x, __nv_bfloat16* __restrict__ xb,
                                               float* __restrict__ ss, int lane) {
  for (int c = 0; c < d / 128; ++c) {
    const int col = c * 128 + lane * 4;
    const uint2 e = *reinterpret_cast<const uint2*>(emb + static_cast<int64_t>(tok) * d + col);
    const __nv_bfloat162 e0 = *reinterpret_cast<const __nv_bfloat162*>(&e.x);
    const __nv_bfloat162 e1 = *reinterpret_cast<const __nv_bfloat162*>(&e.y);
    const float4 v = make_float4(__low2float(e0), __high2float(e0), __low2float(e1), __high2float(e1));
    *reinterpret_cast<float4*>(x + static_cast<int64_t>(r) * d + col) = v;
    *reinterpret_cast<uint2*>(xb + static_cast<int64_t>(r) * d + col) = e;
    float q = (v.x * v.x + v.y * v.y) + (v.z * v.z + v.w * v.w);
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) ss[static_cast<int64_t>(c) * t_stride + r] = q;
  }
}

__device__ __forceinline__ void set_draft_row(LmSlots sl, LmReqState rq, RowsDev rows, int r, int t, int tok) {
  const int slot = rq.slot[r];
  const int pos = sl.len[slot] - 1 + t;
  rows.row_req[r] = r;
  rows.row_pos[r] = pos;
  rows.row_j[r] = t;
  rows.req_first[r] = r;
  rows.req_n[r] = 1;
  rows.req_slot[r] = slot;
  rows.req_pos0[r] = pos;
  rows.row_tok[r] = tok;
}

// Draft step 0 (one warp per row): the step's rows + their embeddings (draft_prep + embed fused).
__global__ void draft_begin_kernel(LmSlots sl, LmReqState rq, RowsDev rows, int n_t, const __nv_bfloat16* emb,
                                   int d, float* x, __nv_bfloat16* xb, float* ss) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *rows.n_rows = n_t;
  if (r >= n_t) return;
  const int slot = rq.slot[r];
  const int tok = sl.tok[static_cast<int64_t>(slot) * sl.max_seq + sl.len[slot] - 1];
  if (lane == 0) set_draft_row(sl, rq, rows, r, 0, tok);
  embed_row_warp(emb, tok, r, d, n_t, x, xb, ss, lane);
}

// After draft step t (one warp per row): argmax_lowest over the LM head's per-tile partials ->
// drafted[r][t]; rows that draft again get step t+1's row and embedding (argmax_reduce +
// draft_post + draft_prep + embed fused into one launch).
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void draft_advance_kernel(LmSlots sl, LmReqState rq, RowsDev rows, const float2* __restrict__ amax,
                                     int n_tiles, int n_t, int t, int n_next, const __nv_bfloat16* emb, int d,
                                     float* x, __nv_bfloat16* xb, float* ss, LaneState ln) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  // overlapped mode: a cancelled step t also cancels t+1 (its rows stay empty)
  if (ln.step_dec && ln.step_dec[t] == 2) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && n_next > 0) ln.step_dec[t + 1] = 2;
    return;
  }
  // decision for step t+1, taken once for the whole grid (first block to get here): cancel it
  // if no request is left on the frontier the verify lane has published so far
  __shared__ int s_dec;
  if (ln.step_dec && n_next > 0) {
    if (threadIdx.x == 0) {
      const int mine = ld_acquire_gpu(ln.alive) == 0 ? 2 : 1;
      const int prev = atomicCAS(&ln.step_dec[t + 1], 0, mine);
      s_dec = prev == 0 ? mine : prev;
    }
    __syncthreads();
  }
  const bool cancel_next = ln.step_dec && n_next > 0 && s_dec == 2;
  if (r >= n_t) return;
  float bv = -3.402823466e38f;
  int bi = 0x7fffffff;
  for (int m = lane; m < n_tiles; m += 32) {
    const float2 p = amax[static_cast<int64_t>(m) * n_t + r];
    const int pi = __float_as_int(p.y);
    if (p.x > bv || (p.x == bv && pi < bi)) {
      bv = p.x;
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
  FASER_DCHECK(static_cast<unsigned>(bi) < kTokLimit, "FASER check: draft_advance row %d t %d argmax %d (n_t %d)\n", r, t,
               bi, n_t);
  if (lane == 0) rq.drafted[r * kMS + t] = bi;
  if (r < n_next) {  // rows are sorted by k' descending: the first n_next rows draft again
    if (cancel_next) {
      if (lane == 0) rows.req_n[r] = 0;  // attention skips the request
    } else {
      if (lane == 0) set_draft_row(sl, rq, rows, r, t + 1, bi);
      embed_row_warp(emb, bi, r, d, n_next, x, xb, ss, lane);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && n_next > 0) *rows.n_rows = cancel_next ? 0 : n_next;
}

// Verify rows' input tokens + their embeddings, one warp per row (verify_tokens + embed fused).
__global__ void verify_begin_kernel(LmSlots sl, LmReqState rq, RowsDev rows, int rows_cap, const __nv_bfloat16* emb,
                                    int d, float* x, __nv_bfloat16* xb, float* ss) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= rows_cap || i >= *rows.n_rows) return;
  const int r = rows.row_req[i], j = rows.row_j[i];
  const int slot = rq.slot[r];
  const int tok = j == 0 ? sl.tok[static_cast<int64_t>(slot) * sl.max_seq + sl.len[slot] - 1]
                         : rq.drafted[r * kMS + j - 1];
  FASER_DCHECK(static_cast<unsigned>(tok) < kTokLimit, "FASER check: verify_begin row %d req %d j %d slot %d token %d\n",
               i, r, j, slot, tok);
  if (lane == 0) rows.row_tok[i] = tok;
  embed_row_warp(emb, tok, i, d, rows_cap, x, xb, ss, lane);
}

// Final argmax_lowest per verify row over the LM head's per-tile partials, written both per row
// and per (request, drafted position) (argmax_reduce + truth_scatter fused), one warp per row.
__global__ void verify_argmax_kernel(RowsDev rows, int n_tiles, int t_stride, const float2* __restrict__ amax,
                                     int* __restrict__ truth, int* __restrict__ truth_rj) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= t_stride || i >= *rows.n_rows) return;
  float bv = -3.402823466e38f;
  int bi = 0x7fffffff;
  for (int m = lane; m < n_tiles; m += 32) {
    const float2 p = amax[static_cast<int64_t>(m) * t_stride + i];
    const int pi = __float_as_int(p.y);
    if (p.x > bv || (p.x == bv && pi < bi)) {
      bv = p.x;
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
  if (lane == 0) {
    truth[i] = bi;
    truth_rj[rows.row_req[i] * kMS + rows.row_j[i]] = bi;
  }
}

__global__ void draft_post_kernel(LmReqState rq, const int* argmax, int n_t, int t) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n_t) rq.drafted[r * kMS + t] = argmax[r];
}

// Row tokens of a verify forward (whole verify or one overlap chunk): row (r, j) reads
// ctx.back() for j == 0, else drafted[r][j-1].
__global__ void verify_tokens_kernel(LmSlots sl, LmReqState rq, RowsDev rows, int rows_cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows_cap || i >= *rows.n_rows) return;
  const int r = rows.row_req[i], j = rows.row_j[i];
  const int slot = rq.slot[r];
  const int tok = j == 0 ? sl.tok[static_cast<int64_t>(slot) * sl.max_seq + sl.len[slot] - 1]
                         : rq.drafted[r * kMS + j - 1];
  FASER_DCHECK(static_cast<unsigned>(tok) < kTokLimit, "FASER check: verify_tokens row %d req %d j %d slot %d token %d\n",
               i, r, j, slot, tok);
  rows.row_tok[i] = tok;
}

// Per-request verify state once every token is drafted: drafted length (EOS stop) and the
// early-exit frontier.
__global__ void verify_init_kernel(LmReqState rq, int n, int layers, int eos) {
  const int r = blockIdx.x;
  if (r >= n) return;
  const int k = rq.k[r];
  for (int j = threadIdx.x; j < kMS; j += blockDim.x) rq.prune_layer[r * kMS + j] = layers;
  if (threadIdx.x == 0) {
    int count = k;
    for (int j = 0; j < k; ++j)
      if (rq.drafted[r * kMS + j] == eos) {  // draft_tokens stops at EOS (sdcore.cpp:56)
        count = j + 1;
        break;
      }
    rq.count[r] = count;
    rq.active[r] = count;
    rq.gate_layers[r] = 0;
    rq.n_pl[r] = 0;
    rq.pr[2 * r] = -1;
    rq.pr[2 * r + 1] = -1;
    rq.failmask[r] = 0u;
  }
}

// Final argmax of every live verify row -> truth_rj[request][j] (chunk-order independent).
__global__ void truth_scatter_kernel(RowsDev rows, const int* __restrict__ argmax, int* __restrict__ truth_rj,
                                     int rows_cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows_cap || i >= *rows.n_rows) return;
  truth_rj[rows.row_req[i] * kMS + rows.row_j[i]] = argmax[i];
}

// K4 fused-estimator prep: each verify row's drafted id d (-1 when the row is off the frontier)
// and W_lm[d] gathered into wg[row] (row 0 of W_lm for rows without a test), so a [128-row block
// x 128] tcgen05 GEMM per block computes z_d in the LM head's own accumulation order.
__global__ void rank_prep_kernel(LmReqState rq, RowsDev rows, const __nv_bfloat16* __restrict__ wlm, int d,
                                 __nv_bfloat16* __restrict__ wg, int* __restrict__ row_d) {
  const int r = blockIdx.x;
  int tok = -1;
  if (r < *rows.n_rows) {
    const int req = rows.row_req[r], j = rows.row_j[r];
    if (j < rq.active[req]) tok = rq.drafted[req * kMS + j];
  }
  FASER_DCHECK(tok < static_cast<int>(kTokLimit), "FASER check: rank prep token %d\n", tok);
  if (threadIdx.x == 0) row_d[r] = tok;
  const uint4* src = reinterpret_cast<const uint4*>(wlm + static_cast<int64_t>(tok < 0 ? 0 : tok) * d);
  uint4* dst = reinterpret_cast<uint4*>(wg + static_cast<int64_t>(r) * d);
  for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = src[i];
}

// K4 fused-estimator decision: sum of the per-tile rank counts of the LM head's kEpiRank epilogue
// (one warp per row) >= k_thr -> the row fails the exit test (exitctl.cpp:56-68).
__global__ void exit_rank_kernel(LmSlots sl, LmReqState rq, RowsDev rows, const int* __restrict__ cnt, int n_tiles,
                                 int t_stride, int k_thr, int rows_cap) {
  const int r = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows_cap || r >= *rows.n_rows) return;
  const int req = rows.row_req[r], j = rows.row_j[r];
  if (j >= rq.active[req]) return;
  const int slot = rq.slot[req];
  if (sl.ncomm[slot] + j == sl.exempt[slot]) return;  // re-entry exemption (sdcore.cpp:118-119)
  int c = 0;
  for (int t = lane; t < n_tiles; t += 32) c += cnt[static_cast<int64_t>(t) * t_stride + r];
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0 && c >= k_thr) atomicOr(&rq.failmask[req], 1u << j);
}

// One thread per request (n <= 1024), single CTA.
// q0: first drafted position of these rows (0, or the chunk start in the overlapped mode, where
// row (i, q0 + jl) sits at local index jl of request i).
// recover = 1 (exempt_rule 2, beyond the reference): the first pruned row keeps running to full
// depth so its final argmax can be committed as the recovery token; rows after it are dropped.
__global__ void frontier_kernel(LmReqState rq, RowsDev rows, int n, int layer, int* src_of, int q0, int recover,
                                int layers) {
  __shared__ int scan[1024];
  const int i = threadIdx.x;
  int keep = 0, old_first = 0, pos0 = 0;
  if (i < n) {
    int act = rq.active[i];
    old_first = rows.req_first[i];
    pos0 = rows.req_pos0[i];
    const int old_n = rows.req_n[i];
    if (act > q0 && old_n > 0) {
      rq.gate_layers[i] += 1;
      const uint32_t live = act >= 32 ? 0xffffffffu : ((1u << act) - 1u);
      const uint32_t f = rq.failmask[i] & live;
      if (f) {
        const int j = __ffs(f) - 1;
        // (recovery mode: the previous recovery row, index act, stops here too)
        const int hi = (recover && rq.pr[2 * i] >= 0) ? act + 1 : act;
        for (int jj = j; jj < hi; ++jj) rq.prune_layer[i * kMS + jj] = layer;
        if (recover) rq.prune_layer[i * kMS + j] = layers;  // runs to full depth
        act = j;
        rq.active[i] = act;
        rq.pr[2 * i] = j;
        rq.pr[2 * i + 1] = layer;
        rq.pl[i * kMS + rq.n_pl[i]] = layer;
        rq.n_pl[i] += 1;
      }
    }
    rq.failmask[i] = 0u;
    keep = act - q0 + ((recover && rq.pr[2 * i] >= 0) ? 1 : 0);  // (+ the recovery row)
    if (q0 == 0 && keep < 1) keep = 1;  // row 0 survives (force-verify, sdcore.cpp:150-166)
    keep = keep < 0 ? 0 : (keep < old_n ? keep : old_n);
  }
  scan[i] = keep;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    const int v = i >= off ? scan[i - off] : 0;
    __syncthreads();
    scan[i] += v;
    __syncthreads();
  }
  const int nf = scan[i] - keep;  // exclusive prefix
  if (i < n) {
    rows.req_first[i] = nf;
    rows.req_n[i] = keep;
    for (int j = 0; j < keep; ++j) {
      src_of[nf + j] = old_first + j;
      rows.row_req[nf + j] = i;
      rows.row_pos[nf + j] = pos0 + j;
      rows.row_j[nf + j] = q0 + j;
    }
  }
  if (i == blockDim.x - 1) *rows.n_rows = scan[i];
}

// Overlapped verify, before chunk q: which requests are still on the frontier, and the chunk's
// rows compacted to theirs (one thread per request, single CTA). Compaction is in place: request
// i's new range starts at or before its old one and no thread reads another request's rows.
__global__ void chunk_frontier_kernel(LmReqState rq, RowsDev rows, int n, int q, int q0, int first, int layers,
                                      int eos, LaneState ln) {
  __shared__ int scan[1024];
  const int i = threadIdx.x;
  int keep = 0, on = 0, pos0 = 0;
  if (i < n) {
    if (first) {  // per-request verify state (the verify_init of the serial path, active = k)
      for (int j = 0; j < kMS; ++j) rq.prune_layer[i * kMS + j] = layers;
      rq.active[i] = rq.k[i];
      rq.gate_layers[i] = 0;
      rq.n_pl[i] = 0;
      rq.pr[2 * i] = -1;
      rq.pr[2 * i + 1] = -1;
      rq.failmask[i] = 0u;
      rq.span[i] = 0;
    }
    const int old_n = rows.req_n[i];
    pos0 = rows.req_pos0[i];
    const int32_t* d = rq.drafted + i * kMS;
    const int32_t* tr = rq.truth_rj + i * kMS;
    bool ok = old_n > 0 && rq.active[i] > q0;
    for (int j = 0; ok && j < q0; ++j) ok = d[j] != eos && d[j] == tr[j];
    if (ok) {
      on = 1;
      keep = old_n;
      for (int j = 0; j < old_n; ++j)
        if (d[q0 + j] == eos) {  // draft_tokens stops at EOS (sdcore.cpp:56): no rows past it
          keep = j + 1;
          break;
        }
      rq.span[i] = q0 + keep;
    }
  }
  const int n_on = __syncthreads_count(on);
  scan[i] = keep;
  __syncthreads();
  for (int off = 1; off < blockDim.x; off <<= 1) {
    const int v = i >= off ? scan[i - off] : 0;
    __syncthreads();
    scan[i] += v;
    __syncthreads();
  }
  const int nf = scan[i] - keep;
  if (i < n) {
    rows.req_first[i] = nf;
    rows.req_n[i] = keep;
    for (int j = 0; j < keep; ++j) {
      rows.row_req[nf + j] = i;
      rows.row_pos[nf + j] = pos0 + j;
      rows.row_j[nf + j] = q0 + j;
    }
  }
  if (i == blockDim.x - 1) {
    *rows.n_rows = scan[i];
    ln.rec[2 * q] = n_on;
    ln.rec[2 * q + 1] = scan[i];
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ln.alive), "r"(n_on) : "memory");
  }
}

__global__ void chunk_finalize_kernel(LmReqState rq, int n, int eos, int nchunks, int chunk, LaneState ln) {
  __shared__ int s_res[kMS + 1];
  const int i = threadIdx.x;
  for (int q = i; q <= kMS; q += blockDim.x) s_res[q] = 0;
  __syncthreads();
  int surv = 0;
  if (i < n) {
    // every draft step has finished when this runs (the last chunk waited for the draft lane):
    // the EOS stop scans all drafted tokens up to the first cancelled step, as the serial path
    const int k = rq.k[i];
    int t_c = k;
    for (int t = 1; t < k; ++t)
      if (ln.step_dec[t] == 2) {
        t_c = t;
        break;
      }
    const int32_t* d = rq.drafted + i * kMS;
    const int32_t* tr = rq.truth_rj + i * kMS;
    const int span = rq.span[i];
    int count = k;
    for (int j = 0; j < t_c; ++j)
      if (d[j] == eos) {
        count = j + 1;
        break;
      }
    const int act = rq.active[i] < count ? rq.active[i] : count;
    rq.count[i] = count;
    rq.active[i] = act;
    bool ok = act >= count && span >= count;
    for (int j = 0; ok && j < count; ++j) ok = d[j] == tr[j];
    surv = ok ? 1 : 0;
    // the frontier ended in the last chunk the request had rows in; unless everything it
    // drafted was accepted, that chunk's verification reset it
    if (!ok && span > 0) atomicAdd(&s_res[(span - 1) / chunk], 1);
  }
  const int ns = __syncthreads_count(surv);
  if (i == 0) ln.rec[2 * nchunks] = ns;
  for (int q = i; q < nchunks; q += blockDim.x) ln.resets[q] = s_res[q];
}

// Compaction, pass 1: copy the surviving rows' residual (fp32 + bf16 operand copy + per-chunk
// sums of squares) to scratch in their new order.
__global__ void gather_kernel(RowsDev rows, const int* __restrict__ src_of, int d, int t_stride,
                              const float* __restrict__ x, const __nv_bfloat16* __restrict__ xb,
                              const float* __restrict__ ss, float* __restrict__ xs,
                              __nv_bfloat16* __restrict__ xbs, float* __restrict__ sss) {
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  const int src = src_of[r];
  const float4* s4 = reinterpret_cast<const float4*>(x + static_cast<int64_t>(src) * d);
  float4* o4 = reinterpret_cast<float4*>(xs + static_cast<int64_t>(r) * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) o4[c] = s4[c];
  const uint4* b4 = reinterpret_cast<const uint4*>(xb + static_cast<int64_t>(src) * d);
  uint4* ob4 = reinterpret_cast<uint4*>(xbs + static_cast<int64_t>(r) * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) ob4[c] = b4[c];
  for (int c = threadIdx.x; c < d / 128; c += blockDim.x)
    sss[static_cast<int64_t>(c) * t_stride + r] = ss[static_cast<int64_t>(c) * t_stride + src];
}

// Compaction, pass 2: scratch -> live buffers.
__global__ void scatter_back_kernel(RowsDev rows, int d, int t_stride, const float* __restrict__ xs,
                                    const __nv_bfloat16* __restrict__ xbs, const float* __restrict__ sss,
                                    float* __restrict__ x, __nv_bfloat16* __restrict__ xb,
                                    float* __restrict__ ss) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int r = blockIdx.x;
  if (r >= *rows.n_rows) return;
  const float4* s4 = reinterpret_cast<const float4*>(xs + static_cast<int64_t>(r) * d);
  float4* o4 = reinterpret_cast<float4*>(x + static_cast<int64_t>(r) * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) o4[c] = s4[c];
  const uint4* b4 = reinterpret_cast<const uint4*>(xbs + static_cast<int64_t>(r) * d);
  uint4* ob4 = reinterpret_cast<uint4*>(xb + static_cast<int64_t>(r) * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) ob4[c] = b4[c];
  for (int c = threadIdx.x; c < d / 128; c += blockDim.x)
    ss[static_cast<int64_t>(c) * t_stride + r] = sss[static_cast<int64_t>(c) * t_stride + r];
}

__global__ void accept_commit_kernel(LmSlots sl, LmReqState rq, RowsDev rows, StepCtl ctl,
                                     faser_round_result* __restrict__ results) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= ctl.n) return;
  const int slot = rq.slot[r];
  const int count = rq.count[r];
  const int L = ctl.layers;
  const bool ee = ctl.early_exit != 0;
  const int32_t* d = rq.drafted + r * kMS;
  const int32_t* plr = rq.prune_layer + r * kMS;
  const int32_t* truth = rq.truth_rj + r * kMS;
  int active = ee ? rq.active[r] : count;
  int pr_j = rq.pr[2 * r], pr_l = rq.pr[2 * r + 1];
  bool pruned = pr_j >= 0;
  faser_round_result* rr = results + rq.live_idx[r];
  faser_verify_outcome& o = rr->outcome;

  int acc = 0, rec = -1;
  bool mismatch = false;
  for (int j = 0; j < active; ++j) {
    if (d[j] == truth[j]) {
      ++acc;
    } else {
      rec = truth[j];
      mismatch = true;
      break;
    }
  }
  const bool recover = ctl.exempt_rule == 2;
  if (recover && pruned && !mismatch && active > 0 && pr_j < count) rec = truth[pr_j];  // the kept row's argmax
  if (ee && active == 0) {  // progress guarantee: force-verify token 0
    if (d[0] == truth[0]) {
      acc = 1;
    } else {
      rec = truth[0];
      mismatch = true;
    }
    if (count > 1) {
      pr_j = 1;
      pr_l = plr[1];
    } else {
      pruned = false;
      pr_j = pr_l = -1;
    }
    active = 1;
  }
  double flr = 0.0;
  if (ee) {
    for (int j = 0; j < count; ++j) flr += (j < active) ? L : plr[j];
  } else {
    flr = static_cast<double>(L) * count;
  }
  o.submitted = count;
  o.accepted_count = acc;
  o.has_recovery = rec >= 0;
  o.recovery_token = rec;
  o.has_pruned = pruned;
  o.pruned_index = pruned ? pr_j : -1;
  o.pruned_layer = pruned ? pr_l : -1;
  o.gate_layers = ee ? rq.gate_layers[r] : 0;
  o.full_layers_run = flr;
  // false_prune needs the full-depth argmax of the pruned row, which a pruned verify never
  // computes (that is the saving); reported as -1 = "not evaluated" on this path.
  o.false_prune = (pruned && !mismatch && acc == pr_j && pr_j < count) ? -1 : 0;
  // recovery mode evaluates the pruned row at full depth: false_prune is exact there
  if (recover && pruned && !mismatch && acc == pr_j && pr_j < count && active > 0)
    o.false_prune = d[pr_j] == truth[pr_j] ? 1 : 0;
  const int npl = ee ? rq.n_pl[r] : 0;
  o.n_prune_layers = npl;
  for (int i = 0; i < npl; ++i) o.prune_layers[i] = rq.pl[r * kMS + i];
  const int base = sl.len[slot];
  o.base_len = base;
  rr->req_id = rq.req_id[r];
  rr->spec_length = rq.spec[r];
  rr->drafted = count;

  // commit (sdcore.cpp:182-197)
  const int ncomm0 = sl.ncomm[slot];
  int done = sl.done[slot];
  int nc = ncomm0, c = 0;
  const int mo = sl.max_out[slot];
  int32_t* out_row = sl.tok + static_cast<int64_t>(slot) * sl.max_seq + base;
  for (int j = 0; j < acc && !done; ++j) {
    out_row[c] = d[j];
    rr->tokens[c++] = d[j];
    ++nc;
    if (d[j] == ctl.eos || nc == mo) done = 1;
  }
  if (rec >= 0 && !done) {
    out_row[c] = rec;
    rr->tokens[c++] = rec;
    ++nc;
    if (rec == ctl.eos || nc == mo) done = 1;
  }
  sl.len[slot] = base + c;
  sl.ncomm[slot] = nc;
  sl.done[slot] = done;
  int ex = sl.exempt[slot];
  if (ctl.exempt_rule == 1) ex = pruned ? ncomm0 + pr_j : -1;
  if (recover) ex = -1;  // the pruned position is resolved by the recovery token
  sl.exempt[slot] = ex;
  rr->done = done;
  rr->exempt_position = ex;
  rr->n_committed_total = nc;
  rr->committed = c;
}

__global__ void ptab_scatter_kernel(int* ptab, int max_pages, const int* tr, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ptab[static_cast<int64_t>(tr[3 * i]) * max_pages + tr[3 * i + 1]] = tr[3 * i + 2];
}

__global__ void admit_kernel(LmSlots sl, const LmAdmit* __restrict__ a, int n) {
  const int e = blockIdx.x;
  if (e >= n) return;
  const LmAdmit ad = a[e];
  int32_t* row = sl.tok + static_cast<int64_t>(ad.slot) * sl.max_seq;
  for (int i = threadIdx.x; i < ad.len; i += blockDim.x) row[i] = ad.src[i];
  if (threadIdx.x == 0) {
    sl.len[ad.slot] = ad.len;
    sl.ncomm[ad.slot] = 0;
    sl.max_out[ad.slot] = ad.max_out;
    sl.done[ad.slot] = 0;
    sl.exempt[ad.slot] = -1;
  }
}

__global__ void prefill_tokens_kernel(LmSlots sl, RowsDev rows, int rows_cap) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_cap || r >= *rows.n_rows) return;
  const int slot = rows.req_slot[rows.row_req[r]];
  rows.row_tok[r] = sl.tok[static_cast<int64_t>(slot) * sl.max_seq + rows.row_pos[r]];
}

inline int cdiv(int a, int b) { return (a + b - 1) / b; }

}  // namespace

cudaError_t lm_draft_prep(LmSlots sl, LmReqState rq, RowsDev rows, int n_t, int t, cudaStream_t s) {
  draft_prep_kernel<<<cdiv(n_t > 0 ? n_t : 1, 256), 256, 0, s>>>(sl, rq, rows, n_t, t);
  return cudaGetLastError();
}
namespace {
template <class K, class... A>
cudaError_t launch_pdl(K kern, int blocks, int threads, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
}  // namespace

cudaError_t lm_draft_begin(LmSlots sl, LmReqState rq, RowsDev rows, int n_t, const __nv_bfloat16* emb, int d,
                           float* x, __nv_bfloat16* xb, float* ss, cudaStream_t s) {
  const int n = n_t > 0 ? n_t : 1;
  return launch_pdl(draft_begin_kernel, cdiv(n * 32, 256), 256, s, sl, rq, rows, n_t, emb, d, x, xb, ss);
}
cudaError_t lm_draft_advance(LmSlots sl, LmReqState rq, RowsDev rows, const float2* amax, int n_tiles, int n_t,
                             int t, int n_next, const __nv_bfloat16* emb, int d, float* x, __nv_bfloat16* xb,
                             float* ss, cudaStream_t s, const LaneState* lane) {
  if (n_t <= 0) return cudaSuccess;
  const LaneState ln = lane ? *lane : LaneState{nullptr, nullptr, nullptr, nullptr};
  return launch_pdl(draft_advance_kernel, cdiv(n_t * 32, 256), 256, s, sl, rq, rows, amax, n_tiles, n_t, t,
                    n_next, emb, d, x, xb, ss, ln);
}
cudaError_t lm_verify_begin(LmSlots sl, LmReqState rq, RowsDev rows, int rows_cap, const __nv_bfloat16* emb, int d,
                            float* x, __nv_bfloat16* xb, float* ss, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  return launch_pdl(verify_begin_kernel, cdiv(rows_cap * 32, 256), 256, s, sl, rq, rows, rows_cap, emb, d, x, xb, ss);
}
cudaError_t lm_verify_argmax(RowsDev rows, int n_tiles, int rows_cap, const float2* amax, int* truth, int* truth_rj,
                             cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  return launch_pdl(verify_argmax_kernel, cdiv(rows_cap * 32, 256), 256, s, rows, n_tiles, rows_cap, amax, truth,
                    truth_rj);
}
cudaError_t lm_draft_post(LmReqState rq, const int* argmax, int n_t, int t, cudaStream_t s) {
  if (n_t <= 0) return cudaSuccess;
  draft_post_kernel<<<cdiv(n_t, 256), 256, 0, s>>>(rq, argmax, n_t, t);
  return cudaGetLastError();
}
cudaError_t lm_verify_tokens(LmSlots sl, LmReqState rq, RowsDev rows, int rows_cap, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  verify_tokens_kernel<<<cdiv(rows_cap, 128), 128, 0, s>>>(sl, rq, rows, rows_cap);
  return cudaGetLastError();
}
cudaError_t lm_verify_init(LmReqState rq, int n, int layers, int eos, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  verify_init_kernel<<<n, 32, 0, s>>>(rq, n, layers, eos);
  return cudaGetLastError();
}
cudaError_t lm_truth_scatter(RowsDev rows, const int* argmax, int* truth_rj, int rows_cap, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  truth_scatter_kernel<<<cdiv(rows_cap, 128), 128, 0, s>>>(rows, argmax, truth_rj, rows_cap);
  return cudaGetLastError();
}
cudaError_t lm_rank_prep(LmReqState rq, RowsDev rows, const __nv_bfloat16* wlm, int d, __nv_bfloat16* wg,
                         int* row_d, int rows_cap, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  if (d % 8) return cudaErrorInvalidValue;
  rank_prep_kernel<<<rows_cap, 128, 0, s>>>(rq, rows, wlm, d, wg, row_d);
  return cudaGetLastError();
}
cudaError_t lm_exit_rank(LmSlots sl, LmReqState rq, RowsDev rows, const int* cnt, int n_tiles, int t_stride,
                         int k_thr, int rows_cap, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  exit_rank_kernel<<<cdiv(rows_cap, 4), 128, 0, s>>>(sl, rq, rows, cnt, n_tiles, t_stride, k_thr, rows_cap);
  return cudaGetLastError();
}
cudaError_t lm_frontier_compact(LmSlots sl, LmReqState rq, RowsDev rows, int n, int layer,
                                int* src_of, cudaStream_t s, int q0, int recover, int layers) {
  (void)sl;
  if (n <= 0) return cudaSuccess;
  if (n > 1024) return cudaErrorInvalidValue;
  frontier_kernel<<<1, cdiv(n, 32) * 32, 0, s>>>(rq, rows, n, layer, src_of, q0, recover, layers);
  return cudaGetLastError();
}
cudaError_t lm_chunk_frontier(LmReqState rq, RowsDev rows, int n, int q, int q0, int first, int layers, int eos,
                              LaneState lane, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > 1024) return cudaErrorInvalidValue;
  chunk_frontier_kernel<<<1, cdiv(n, 32) * 32, 0, s>>>(rq, rows, n, q, q0, first, layers, eos, lane);
  return cudaGetLastError();
}
cudaError_t lm_chunk_finalize(LmReqState rq, int n, int eos, int nchunks, int chunk, LaneState lane, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n > 1024 || chunk < 1 || nchunks > kMS) return cudaErrorInvalidValue;
  chunk_finalize_kernel<<<1, cdiv(n, 32) * 32, 0, s>>>(rq, n, eos, nchunks, chunk, lane);
  return cudaGetLastError();
}
cudaError_t lm_gather_rows(RowsDev rows, const int* src_of, int d, int t_stride, float* x,
                           __nv_bfloat16* xb, float* ss, float* xs, __nv_bfloat16* xbs, float* sss,
                           cudaStream_t s) {
  if (t_stride <= 0) return cudaSuccess;
  gather_kernel<<<t_stride, 256, 0, s>>>(rows, src_of, d, t_stride, x, xb, ss, xs, xbs, sss);
  scatter_back_kernel<<<t_stride, 256, 0, s>>>(rows, d, t_stride, xs, xbs, sss, x, xb, ss);
  return cudaGetLastError();
}
cudaError_t lm_accept_commit(LmSlots sl, LmReqState rq, RowsDev rows, StepCtl ctl,
                             faser_round_result* results, cudaStream_t s) {
  if (ctl.n <= 0) return cudaSuccess;
  accept_commit_kernel<<<cdiv(ctl.n, 64), 64, 0, s>>>(sl, rq, rows, ctl, results);
  return cudaGetLastError();
}
cudaError_t lm_ptab_scatter(int* ptab, int max_pages, const int* triples, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  ptab_scatter_kernel<<<cdiv(n, 256), 256, 0, s>>>(ptab, max_pages, triples, n);
  return cudaGetLastError();
}
cudaError_t lm_admit(LmSlots sl, const LmAdmit* admits, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  admit_kernel<<<n, 128, 0, s>>>(sl, admits, n);
  return cudaGetLastError();
}
cudaError_t lm_prefill_tokens(LmSlots sl, RowsDev rows, int rows_cap, cudaStream_t s) {
  if (rows_cap <= 0) return cudaSuccess;
  prefill_tokens_kernel<<<cdiv(rows_cap, 256), 256, 0, s>>>(sl, rows, rows_cap);
  return cudaGetLastError();
}

}  // namespace faser

// toy_kernels.cuh — device-side state layout + launchers for the toy-model path (configs 1-2).
//
// The reference's toy pair (toylm.cpp) is a pure function of the context, so the "KV cache"
// of a request is three 64-bit running hash states: hash_tokens(noise_seed, ctx),
// hash_tokens(mix_seed, ctx) (rng.hpp:28-32) and the last `order` tokens (read from the
// token row). Appending a token is O(1) (one hash_combine), rollback is "keep the state at
// the accepted length" — the same shape as a paged-KV append/rollback, minus the bytes.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "faser/engine.h"

namespace faser {

constexpr int kMaxBatchHW = 1024;  // hard cap on slots per engine (StepIn arrays)

struct ToyDev {
  uint64_t table_seed, noise_seed, mix_seed;
  double divergence, logit_scale, noise_scale;
  int32_t vocab, layers, order, eos;
};

// Per-slot request state, structure-of-arrays in HBM.
struct SlotState {
  int32_t* tok;       // [slots][max_seq] prompt ++ committed
  int32_t* len;       // [slots] context length
  int32_t* ncomm;     // [slots] |committed|
  int32_t* max_out;   // [slots]
  int32_t* done;      // [slots]
  int32_t* exempt;    // [slots] exempt_position (-1 unset)
  uint64_t* nh;       // [slots] hash_tokens(noise_seed, ctx)
  uint64_t* mh;       // [slots] hash_tokens(mix_seed, ctx)
  int32_t* draft;     // [slots][FASER_MAX_SPEC] drafted tokens of the current round
  int32_t* draft_len; // [slots]
  uint64_t* mh_at;    // [slots][FASER_MAX_SPEC+1] mix-hash state at ctx ++ d[0..j)
  int32_t max_seq;
};

struct AdmitEntry {
  const int32_t* src;  // device copy of the context (prompt ++ committed)
  int32_t slot, len, max_out, ncomm, exempt, reserved;
};

// Round inputs uploaded once per step (one H2D from pinned memory). Packed: the fixed
// header is followed by n_live live slots, n_live k_i, n_live request ids and n_admit
// admission entries, so the copy is ~16 B per live request instead of a fixed table.
struct StepIn {
  int32_t n_live;
  int32_t n_admit;
  int32_t early_exit;  // 0 full_verify, 1 verify_with_early_exit
  int32_t gate_lo;     // first gated layer (inclusive), already max(first,1)
  int32_t gate_hi;     // min(stop, L) (exclusive); gate inactive => lo >= hi
  int32_t commit;      // 1: apply SpeculativeEngine::commit + exempt rule
  int32_t exempt_rule;
  int32_t total_bytes;
  int32_t off_live_slot, off_k, off_req_id, off_admit;  // byte offsets from `this`
  int32_t off_tok;  // admitted prompts, concatenated (AdmitEntry::src may point here on the device)
  int32_t k_table[FASER_MAX_LAYERS + 1];

  __host__ __device__ const char* base() const { return reinterpret_cast<const char*>(this); }
  __host__ __device__ char* base() { return reinterpret_cast<char*>(this); }
  __host__ __device__ const int32_t* live_slot() const { return reinterpret_cast<const int32_t*>(base() + off_live_slot); }
  __host__ __device__ const int32_t* k() const { return reinterpret_cast<const int32_t*>(base() + off_k); }
  __host__ __device__ const int64_t* req_id() const { return reinterpret_cast<const int64_t*>(base() + off_req_id); }
  __host__ __device__ const AdmitEntry* admit() const { return reinterpret_cast<const AdmitEntry*>(base() + off_admit); }
  __host__ __device__ int32_t* live_slot() { return reinterpret_cast<int32_t*>(base() + off_live_slot); }
  __host__ __device__ int32_t* k() { return reinterpret_cast<int32_t*>(base() + off_k); }
  __host__ __device__ int64_t* req_id() { return reinterpret_cast<int64_t*>(base() + off_req_id); }
  __host__ __device__ AdmitEntry* admit() { return reinterpret_cast<AdmitEntry*>(base() + off_admit); }
  __host__ __device__ int32_t* tok() { return reinterpret_cast<int32_t*>(base() + off_tok); }

  // Lays out the arrays for (n_live, n_admit, prompt tokens carried inline); returns total bytes.
  __host__ int32_t layout(int32_t live, int32_t admits, int32_t tokens = 0) {
    auto al = [](int32_t x, int32_t a) { return (x + a - 1) / a * a; };
    n_live = live;
    n_admit = admits;
    off_live_slot = al(static_cast<int32_t>(sizeof(StepIn)), 16);
    off_k = off_live_slot + 4 * live;
    off_req_id = al(off_k + 4 * live, 8);
    off_admit = al(off_req_id + 8 * live, 16);
    off_tok = al(off_admit + static_cast<int32_t>(sizeof(AdmitEntry)) * admits, 16);
    total_bytes = off_tok + 4 * tokens;
    return total_bytes;
  }
  static constexpr size_t capacity(int32_t max_live, int64_t max_tokens = 0) {
    return sizeof(StepIn) + 96 + static_cast<size_t>(max_live) * (4 + 4 + 8 + sizeof(AdmitEntry)) +
           4 * static_cast<size_t>(max_tokens);
  }
};

// Launchers (all asynchronous on `stream`). Return cudaGetLastError().
cudaError_t toy_admit(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_admit,
                      cudaStream_t stream);
cudaError_t toy_draft(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_live,
                      cudaStream_t stream);
cudaError_t toy_verify_commit(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_live,
                              faser_round_result* results, cudaStream_t stream);
// draft (warp 0 of block p) + verify + commit of request p in one launch (the engine's step)
cudaError_t toy_draft_verify_commit(const ToyDev& m, SlotState st, const StepIn* in_dev, int n_live,
                                    faser_round_result* results, cudaStream_t stream);
// Row ops for the stateless API: op 0 final_and_noise, 1 target_logits(layers), 2 target_next,
// 3 draft_next.
cudaError_t toy_rows(const ToyDev& m, int op, int n, const int32_t* tokens, const int64_t* off,
                     const int32_t* layers, double* z0, double* z1, int32_t* out,
                     cudaStream_t stream);

bool toy_vocab_supported(int vocab);

}  // namespace faser

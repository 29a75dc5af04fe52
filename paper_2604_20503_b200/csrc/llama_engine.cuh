// llama_engine.cuh — the Llama-style serving engine behind faser_engine (model kind LLAMA).
#pragma once
#include <cstdint>

#include "faser/engine.h"

namespace faser {

class LlamaEngine;

// All functions throw faser::Fail-like errors via the status/message pair.
struct LmStatus {
  faser_status st = FASER_OK;
  const char* msg = "";
};

LlamaEngine* llama_engine_create(const faser_model_desc* model, const faser_engine_cfg* cfg,
                                 faser_status* st, const char** msg);
void llama_engine_destroy(LlamaEngine* e);
const char* llama_last_error(const LlamaEngine* e);

faser_status llama_submit(LlamaEngine* e, int64_t req_id, const int32_t* prompt, int32_t len,
                          int32_t max_out);
faser_status llama_set_spec_lengths(LlamaEngine* e, const int64_t* ids, const int32_t* k, int32_t n);
faser_status llama_live_requests(LlamaEngine* e, int64_t* ids, int32_t cap, int32_t* n);
faser_status llama_step(LlamaEngine* e, const faser_step_plan* plan, faser_round_result* out,
                        int32_t cap, int32_t* n_out);
faser_status llama_get_committed(LlamaEngine* e, int64_t req_id, int32_t* buf, int32_t cap, int32_t* n);
faser_status llama_release(LlamaEngine* e, int64_t req_id);
int32_t llama_pending_work(const LlamaEngine* e);
void llama_last_step_timing(const LlamaEngine* e, float* d, float* v, float* s);
float llama_last_step_prefill(const LlamaEngine* e);
faser_status llama_join_lanes(LlamaEngine* e);
faser_status llama_set_prefill_lane(LlamaEngine* e, int on);
faser_status llama_set_skip_mask(LlamaEngine* e, int mask);
faser_status llama_set_sampling(LlamaEngine* e, double temperature, uint64_t seed);
void llama_last_step_bytes(const LlamaEngine* e, int64_t* h2d, int64_t* d2h);
void* llama_stream(const LlamaEngine* e);
faser_status llama_last_timeline(const LlamaEngine* e, faser_timeline_event* ev, int32_t cap, faser_timeline_info* info);
int64_t llama_launches(const LlamaEngine* e);
faser_status llama_debug_verify_logits(LlamaEngine* e, int32_t stage, float* logits, int64_t* row_ids,
                                       int32_t cap_rows, int32_t* rows);
faser_status llama_debug_drafted(LlamaEngine* e, int32_t* drafted, int32_t cap, int32_t* n);
faser_status llama_debug_weights(LlamaEngine* e, int32_t model, int32_t which, int32_t layer, int64_t offset,
                                 int32_t n, uint16_t* out);
faser_status llama_set_kernel_timing(LlamaEngine* e, int32_t on);
faser_status llama_kernel_stats(LlamaEngine* e, int32_t cls, double* ms, int64_t* launches, double* bytes);
faser_status llama_kernel_flops(LlamaEngine* e, int32_t cls, double* flops);
faser_status llama_debug_kv_pages(LlamaEngine* e, int64_t req_id, int32_t* pages, int32_t cap, int32_t* n);

}  // namespace faser

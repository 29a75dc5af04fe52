/*
 * faser/engine.h — C ABI of the B200-native FASER speculative-decoding data path.
 *
 * The reference (`/root/reference/proj/core`, C++20, CPU only) exposes the path as an
 * in-process C++ class API. Every entry point below names the reference interface it
 * replaces (file:line). Conventions:
 *   - plain pointers + sizes, caller-owned HOST buffers unless a name says `_dev`;
 *   - reference exceptions map to status codes (std::invalid_argument -> FASER_EINVAL,
 *     std::logic_error -> FASER_EILLEGAL_STATE, errors.hpp:8-18 -> ECONFIG/EPARSE/EFIT);
 *   - the message of the mapped exception is returned by faser_last_error();
 *   - the library never falls back to CPU: if the CUDA kernels cannot run the call fails
 *     with FASER_ECUDA.
 */
#ifndef FASER_ENGINE_H
#define FASER_ENGINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FASER_ABI_VERSION 3
/* Largest speculative length a request may be assigned in one round (S = {1..10} in the
 * reference, drafter.hpp:16). Bounds per-request outcome arrays. */
#define FASER_MAX_SPEC 32
/* Largest layer count the per-layer exit-threshold table covers. */
#define FASER_MAX_LAYERS 128

typedef enum faser_status {
  FASER_OK = 0,
  FASER_EINVAL = 1,         /* std::invalid_argument */
  FASER_EILLEGAL_STATE = 2, /* std::logic_error: draft/commit on done request, stale outcome */
  FASER_ECONFIG = 3,        /* specsim::ConfigError */
  FASER_EPARSE = 4,         /* specsim::ParseError */
  FASER_EFIT = 5,           /* specsim::FitError */
  FASER_ECUDA = 6,          /* device missing / kernel failure (never silently degraded) */
  FASER_ENCCL = 7,
  FASER_ENOMEM = 8,
  FASER_ECAPACITY = 9       /* engine slot / sequence capacity exceeded */
} faser_status;

/* ---------------------------------------------------------------- model descriptors */

/* LayeredToyLM::Params (toylm.hpp:42-51). `divergence` is eta of draft_next. */
typedef struct faser_toy_params {
  uint64_t seed;
  int32_t vocab;
  int32_t layers;
  int32_t order;
  int32_t reserved0;
  double divergence;
  uint64_t noise_seed;
  double logit_scale;
  double noise_scale;
} faser_toy_params;

/* ExitPolicy (exitctl.hpp:14-22). */
typedef struct faser_exit_policy {
  int32_t l_init;
  int32_t k_init;
  int32_t k_final;
} faser_exit_policy;

/* GatePlan (exitctl.hpp:60-67): gated layers are [first_layer, stop_layer). */
typedef struct faser_gate_plan {
  int32_t first_layer;
  int32_t stop_layer;
  double s_eff;
} faser_gate_plan;

/* GateEntry (exitctl.hpp:24-28). */
typedef struct faser_gate_entry {
  int32_t spec_length;
  int32_t reserved0;
  double accept_estimate;
} faser_gate_entry;

/* OverlapPlan (overlap.hpp:11-17). */
typedef struct faser_overlap_plan {
  int32_t enabled;
  int32_t chunk;
  double r;
  double predicted_ms;
  double serial_ms;
} faser_overlap_plan;

/* PiecewiseLatencyParams (latmodel.hpp:32-38); stage: 0 draft, 1 target, 2 ee_check, 3 prune. */
typedef struct faser_latency_params {
  int32_t stage;
  int32_t reserved0;
  double knee, a1, gamma1, a2, gamma2, c0, c1, c2;
} faser_latency_params;

/* LatencyModel (latmodel.hpp:92-113). */
typedef struct faser_latency_model {
  faser_latency_params draft, target, ee_check, prune;
} faser_latency_model;

/* VerifyOutcome (sdcore.hpp:59-77), flattened: optionals become has_* flags. */
typedef struct faser_verify_outcome {
  int32_t submitted;
  int32_t accepted_count;
  int32_t has_recovery;
  int32_t recovery_token;
  int32_t has_pruned;
  int32_t pruned_index; /* pruned_at->first  */
  int32_t pruned_layer; /* pruned_at->second */
  int32_t gate_layers;
  double full_layers_run;
  int32_t false_prune;
  int32_t n_prune_layers;
  int32_t prune_layers[FASER_MAX_SPEC];
  int64_t base_len;
} faser_verify_outcome;

/* ------------------------------------------------- stateless batched toy-model kernels
 * Ragged batch convention: request i's context (prompt ++ committed) is
 * tokens[offsets[i] .. offsets[i+1]), offsets has n+1 entries. */

/* LayeredToyLM::final_and_noise (toylm.cpp:42-54) per row -> z_final/z_noise [n][vocab]. */
faser_status faser_toy_final_and_noise(const faser_toy_params* model, int32_t n,
                                       const int32_t* tokens, const int64_t* offsets,
                                       double* z_final, double* z_noise);

/* LayeredToyLM::target_logits (toylm.cpp:56-67) per row at layers[i] -> z [n][vocab]. */
faser_status faser_toy_target_logits(const faser_toy_params* model, int32_t n,
                                     const int32_t* tokens, const int64_t* offsets,
                                     const int32_t* layers, double* z);

/* LayeredToyLM::target_next / draft_next (toylm.cpp:69-85) per row -> out[n]. */
faser_status faser_toy_target_next(const faser_toy_params* model, int32_t n,
                                   const int32_t* tokens, const int64_t* offsets, int32_t* out);
faser_status faser_toy_draft_next(const faser_toy_params* model, int32_t n,
                                  const int32_t* tokens, const int64_t* offsets, int32_t* out);

/* SpeculativeEngine::draft_tokens (sdcore.cpp:45-59) per request.
 * s[i] >= 1, remaining[i] = max_out - |committed| >= 1 (else EILLEGAL_STATE, "done").
 * out [n][FASER_MAX_SPEC], out_len[n]. */
faser_status faser_toy_draft_tokens(const faser_toy_params* model, int32_t n,
                                    const int32_t* tokens, const int64_t* offsets,
                                    const int32_t* s, const int32_t* remaining,
                                    int32_t* out, int32_t* out_len);

/* SpeculativeEngine::full_verify (sdcore.cpp:61-81) when gate == NULL, else
 * SpeculativeEngine::verify_with_early_exit (sdcore.cpp:83-180) with `policy`/`gate`.
 * committed_len[i] = |req.committed| (for exempt positions), exempt[i] = req.exempt_position.
 * k_table (may be NULL) overrides policy->k_at: k_table[layer] for layer in [0, layers]. */
faser_status faser_toy_verify(const faser_toy_params* model, int32_t n, const int32_t* tokens,
                              const int64_t* offsets, const int32_t* committed_len,
                              const int32_t* exempt, const int32_t* drafted,
                              const int32_t* drafted_len, const faser_exit_policy* policy,
                              const faser_gate_plan* gate, faser_verify_outcome* out);

/* ------------------------------------------------------------ stateful serving engine
 * Replaces the missing serving loop's use of SpeculativeEngine + Request (sdcore.hpp:39-116,
 * SPEC.md:541-563): requests are submitted (iteration-boundary admission), every
 * faser_step() runs draft -> verify(+early exit) -> accept -> commit for all live requests
 * on the GPU and returns one faser_round_result per live request. */

enum { FASER_MODEL_TOY = 0, FASER_MODEL_LLAMA = 1 };
/* AblationMode (config.hpp:16). */
enum { FASER_MODE_VSD = 0, FASER_MODE_VSD_AD = 1, FASER_MODE_VSD_AD_EE = 2, FASER_MODE_FULL = 3 };

/* Llama-style random-init bf16 model (configs 3-5; no reference implementation exists, see
 * SURVEY.md section 8c). Weights are a pure function of (seed, tensor, index), regenerated
 * bit-identically by the CPU oracle (oracle/llama_oracle.c). bigram_scale / embed_noise set
 * the acceptance-tunable construction (embedding(t) = bigram_scale * W_lm[g(t)] + noise). */
typedef struct faser_llama_shape {
  int32_t d_model, layers, n_heads, n_kv_heads, head_dim, ffn, vocab, reserved0;
  double rope_theta, rms_eps;
  double bigram_scale, embed_noise, init_std;
  /* fraction of "hard" tokens t whose successor in THIS model is g(t) + V/2 (mod V) instead of
   * g(t): set on the target only, it makes the pair disagree exactly on those contexts and the
   * disagreement is visible from the first layers (early exit has signal). 0 = plain bigram. */
  double hard_fraction;
  uint64_t seed;
} faser_llama_shape;

typedef struct faser_model_desc {
  int32_t kind; /* FASER_MODEL_TOY or FASER_MODEL_LLAMA */
  int32_t reserved0;
  faser_toy_params toy;       /* FASER_MODEL_TOY */
  faser_llama_shape draft;    /* FASER_MODEL_LLAMA */
  faser_llama_shape target;   /* FASER_MODEL_LLAMA */
  uint32_t bigram_a, bigram_b; /* successor map g(t) = (a*t + b) mod vocab shared by both */
} faser_model_desc;

typedef struct faser_engine_cfg {
  int32_t device;
  int32_t max_batch;       /* B_max, config.hpp:50 (256) */
  int32_t max_seq_len;     /* prompt + max_out capacity per request */
  int32_t mode;            /* FASER_MODE_*: EE modes use verify_with_early_exit */
  int32_t default_spec_length; /* fixed_spec_len, config.hpp:51 (4) */
  int32_t exempt_rule;     /* 1: exempt = committed_before + pruned_at.first for one round;
                              2 (LLAMA, EE modes except FULL; beyond the reference's semantics):
                              recovery on prune - the first pruned row keeps running to full depth
                              and its final argmax is committed as the recovery token after a clean
                              prune (still greedy-lossless), no exemption; false_prune is exact */
  faser_exit_policy exit_policy;
  int32_t max_pending;     /* capacity of the submitted-not-admitted queue */
  int32_t pending_tokens;  /* device staging arena for submitted prompts (tokens) */
  int32_t max_spec_length; /* LLAMA: largest k_i a step may use (verify row capacity); 0 = 16 */
  int32_t prefill_rows;    /* LLAMA: rows per prefill forward chunk; 0 = 8192 */
  int32_t debug_capture;   /* LLAMA: 1 = keep per-stage logits of the last step for validation */
  int32_t prefill_lane;    /* LLAMA: 1 = newly admitted requests are prefilled on a side stream
                              (lower priority, own activations) concurrently with the running
                              batch's draft + verify, and join the batch at the next step (not
                              with TP, FULL mode or debug_capture); 0 = admission + prefill +
                              draft + verify in the admission step */
  /* Tensor-parallel verification (config 5): the TARGET is split over tp_size
   * ranks (column-parallel QKV / gate-up, row-parallel O / down + all-reduce, vocab-parallel LM
   * head + all-gathered argmax); the draft is replicated. tp_size <= 1: no TP. Modes VSD and
   * VSD_AD only. Every rank drives its own engine with the same submits and plans. Heads and
   * ffn / 64 must divide by tp_size; the vocabulary need not (each rank's LM-head shard is
   * ceil(vocab / tp_size) rounded up to 128 rows, the padding masked out of the argmax). */
  int32_t tp_size;
  int32_t tp_rank;
  struct faser_tp_group* tp_group; /* from faser_tp_*_group_create; not owned by the engine */
} faser_engine_cfg;

typedef struct faser_step_plan {
  faser_gate_plan gate;         /* used in EE modes; inactive gate == full verify semantics */
  int32_t use_k_table;          /* 1: k_table[layer] replaces exit_policy.k_at */
  int32_t k_table[FASER_MAX_LAYERS + 1];
  faser_overlap_plan overlap;   /* FULL mode: chunked draft/verify co-execution. With
                                   overlap.r in (0,1) the draft lane runs on a green-context
                                   partition of round8(r * SMs) SMs and the verify lane on the
                                   rest; chunk == k runs the two stages back to back on their
                                   partitions (per-share stage profiling). */
  int32_t lane_mode;            /* 0: lanes overlap (verify chunk q || draft chunk q+1);
                                   1: isolated - the same partitions and chunks, serialised (draft
                                   chunk q+1 waits for verify chunk q), the interference baseline */
  int32_t reserved_lane;
} faser_step_plan;

typedef struct faser_round_result {
  int64_t req_id;
  int32_t spec_length;       /* k_i used this round */
  int32_t drafted;           /* tokens drafted (<= k_i: budget / EOS stop) */
  faser_verify_outcome outcome;
  int32_t committed;         /* tokens committed this round (SpeculativeEngine::commit) */
  int32_t done;
  int32_t exempt_position;   /* value for the next round */
  int32_t n_committed_total;
  int32_t tokens[FASER_MAX_SPEC + 1]; /* the tokens committed this round */
} faser_round_result;

typedef struct faser_engine faser_engine;

/* ---- tensor-parallel groups (no reference counterpart: SPEC.md:8 puts TP out of the
 * simulator's scope; the paper ran TP=2 inside vLLM) */
typedef struct faser_tp_group faser_tp_group;
/* NCCL group, one process per GPU: rank 0 makes the 128-byte id, every rank joins with it. */
faser_status faser_tp_nccl_unique_id(uint8_t* id128);
faser_status faser_tp_nccl_group_create(const uint8_t* id128, int32_t size, int32_t rank, int32_t device,
                                        faser_tp_group** out);
/* In-process group on ONE device: the ranks' engines are driven from `size` host threads
 * (single-GPU validation backend of the sharded math). */
faser_status faser_tp_local_group_create(int32_t size, faser_tp_group** out);
void faser_tp_group_destroy(faser_tp_group* g);

faser_status faser_engine_create(const faser_model_desc* model, const faser_engine_cfg* cfg,
                                 faser_engine** out);
void faser_engine_destroy(faser_engine* e);
/* Message of the last failing call on `e` (or of the last failed create when e == NULL). */
const char* faser_last_error(const faser_engine* e);

faser_status faser_submit(faser_engine* e, int64_t req_id, const int32_t* prompt, int32_t len,
                          int32_t max_out);
/* Controller -> engine (AdaptiveDrafter::assign_lengths output, drafter.hpp:105-107). */
faser_status faser_set_spec_lengths(faser_engine* e, const int64_t* req_ids, const int32_t* k,
                                    int32_t n);
/* Requests that the next faser_step() will run, in batch order (admits pending ones). */
faser_status faser_live_requests(faser_engine* e, int64_t* req_ids, int32_t cap, int32_t* n);
faser_status faser_step(faser_engine* e, const faser_step_plan* plan, faser_round_result* out,
                        int32_t cap, int32_t* n_out);
faser_status faser_get_committed(faser_engine* e, int64_t req_id, int32_t* buf, int32_t cap,
                                 int32_t* n);
/* Drops a finished request's host state (its slot is already free once done). */
faser_status faser_release(faser_engine* e, int64_t req_id);
/* Number of live + pending requests. */
int32_t faser_pending_work(const faser_engine* e);
/* Device time (ms, CUDA events on the engine stream) of the last faser_step: draft lane,
 * verify lane and whole step. (Toy engine: admission, draft, verify and commit run as one
 * launch per round, so draft_ms is 0 and verify_ms is the round.) */
faser_status faser_last_step_timing(const faser_engine* e, float* draft_ms, float* verify_ms,
                                    float* step_ms);
/* Switches the admission-prefill lane of an engine created with prefill_lane = 1 off (0: the
 * next step drains it and admissions are prefilled in-step again) or back on (1). */
faser_status faser_set_prefill_lane(faser_engine* e, int32_t on);
/* Sampling acceptance (north-star K6 "greedy/rejection-sampling"; beyond the reference, which is
 * greedy only, sdcore.cpp:61-80). temperature > 0 (LLAMA engines, every mode but
 * FULL): the draft and the target LM heads sample with coupled Gumbel-max noise - the token at
 * absolute position p of request id r is argmax_v(z_v / temperature + G(seed, r, p, v)) for both
 * models - and the greedy match-and-commit kernel (K5) accepts drafted tokens while they equal
 * the target's sample, committing the target's sample at the first mismatch. Every committed
 * token is the target's sample of softmax(z / temperature) given its prefix: lossless in
 * distribution, and identical to non-speculative sampling with the same noise whatever the
 * drafter or k_i (drafter-invariant). In EE modes the fused exit-test estimator ranks the drafted
 * token among the perturbed intermediate values (same noise). temperature 0 restores greedy.
 * Takes effect at the next step; EINVAL for toy engines, FULL mode, or temperature < 0. */
faser_status faser_set_sampling(faser_engine* e, double temperature, uint64_t seed);
/* The serving loop of the missing sim.cpp as one call, for hosts that drive the
 * engine without per-step callbacks: up to n_rounds iterations of
 *   live requests -> k_i = sched_k(seed, req_id - id_base, rounds served so far) over the drafter
 *   candidates -> faser_set_spec_lengths -> (EE modes) make_gate_plan(policy, (k_i, accept_est),
 *   b = live, r) -> faser_step,
 * stopping early when nothing is live. Reports committed tokens and executed rounds. */
faser_status faser_serve_rounds(faser_engine* e, int32_t n_rounds, uint64_t seed, int64_t id_base,
                                const faser_exit_policy* policy, double accept_est, double r, int32_t num_layers,
                                int64_t* tokens_out, int32_t* rounds_out);
/* Timing experiments only (results become invalid): kernel classes the following steps skip,
 * bitmask 1 attention, 2 qkv, 4 o, 8 gate/up, 16 down of the target verify forward (+ 32: of the
 * prefill forwards instead); -1 restores FASER_SKIP. The bench derives in-stream class costs
 * from the verify time with and without a class. */
faser_status faser_debug_set_skip_mask(faser_engine* e, int32_t mask);
/* Makes the engine stream wait for every side lane's enqueued work (the admission-prefill lane),
 * so an event recorded on faser_engine_stream afterwards covers it. */
faser_status faser_engine_join_lanes(faser_engine* e);
/* Part of the last step's draft-lane time spent on admissions + their prefill forwards (ms,
 * from the step start; 0 for the toy engine). */
faser_status faser_last_step_prefill(const faser_engine* e, float* prefill_ms);
/* Bytes the last faser_step copied host->device (step plan + admissions) and
 * device->host (round results). */
faser_status faser_last_step_bytes(const faser_engine* e, int64_t* h2d, int64_t* d2h);
/* PipelineTimeline (overlap.hpp:19-56) of the last overlapped (FULL) step, measured: CUDA events
 * on the two lanes, times in ms from the step's start. Kinds follow TimelineEvent::Kind. */
enum { FASER_EV_DRAFT_CHUNK = 0, FASER_EV_VERIFY_CHUNK = 1, FASER_EV_RESET = 2, FASER_EV_COMMIT = 3 };
typedef struct faser_timeline_event {
  int32_t kind;
  int32_t chunk;
  double start_ms;
  double end_ms;
} faser_timeline_event;
typedef struct faser_timeline_info {
  int32_t n_events;
  int32_t n_chunks;
  int32_t draft_sms;          /* SMs of the draft partition (green context) */
  int32_t verify_sms;         /* SMs of the verify partition */
  int32_t green;              /* 1: green-context partitions, 0: plain concurrent streams */
  int32_t cancelled_draft_steps; /* draft steps cancelled after every frontier was reset */
  int32_t lane_mode;
  int32_t survivors;          /* requests whose every drafted token was verified and accepted */
  /* per chunk q: requests on the frontier with rows in q, its verify rows, and the requests
   * whose frontier was reset by q's verification (rejection or prune: later chunks cancelled) */
  int32_t chunk_alive[FASER_MAX_SPEC + 1];
  int32_t chunk_rows[FASER_MAX_SPEC + 1];
  int32_t chunk_resets[FASER_MAX_SPEC + 1];
  int32_t reserved0;
  double makespan_ms, draft_busy_ms, verify_busy_ms;
  double wasted_draft_ms;     /* draft chunks no request was left to verify */
} faser_timeline_info;
/* Events of the last step into ev[0 .. min(n_events, cap)); FASER_EINVAL if the last step was not
 * an overlapped Llama step. */
faser_status faser_last_timeline(const faser_engine* e, faser_timeline_event* ev, int32_t cap,
                                 faser_timeline_info* info);
/* The engine's CUDA stream (cudaStream_t) so a caller can record events around steps. */
void* faser_engine_stream(const faser_engine* e);
/* Kernel launches issued by this engine since creation (evidence counter). */
int64_t faser_kernel_launches(const faser_engine* e);

/* LLAMA validation mode (cfg.debug_capture = 1): logits of the last step's verify forward.
 * stage = 0: final logits of the surviving rows; stage = l (1..L-1): the gated-layer logits
 * (LM head on RMSNorm of the layer-l residual) of the rows tested at layer l.
 * Writes min(rows, cap_rows) rows of `vocab` floats and, per row, (req_id, j) into row_ids
 * [2*rows] (row j of a request predicts its drafted[j]). Returns the row count in *rows and
 * FASER_EINVAL if the stage was not evaluated in the last step. */
faser_status faser_debug_verify_logits(faser_engine* e, int32_t stage, float* logits,
                                       int64_t* row_ids, int32_t cap_rows, int32_t* rows);
/* Drafted tokens of the last step per live request (batch order), [n][FASER_MAX_SPEC]. */
faser_status faser_debug_drafted(faser_engine* e, int32_t* drafted, int32_t cap, int32_t* n);
/* Page table row of a live request: KV page ids backing positions [0, 64*n). */
faser_status faser_debug_kv_pages(faser_engine* e, int64_t req_id, int32_t* pages, int32_t cap,
                                  int32_t* n);

/* Raw bf16 weight elements [offset, offset+n) of a LLAMA engine's model (0 draft, 1 target),
 * tensor which: 0 lm_head [V][d], 1 embedding [V][d], 2 wqkv, 3 wo, 4 wgu (interleaved), 5 wd
 * of `layer`. For checking the device generator against the oracle's. */
faser_status faser_debug_weights(faser_engine* e, int32_t model, int32_t which, int32_t layer,
                                 int64_t offset, int32_t n, uint16_t* out);

/* Per-kernel-class device timing (CUDA events recorded around every launch of the class on its
 * stream; enabled by faser_set_kernel_timing, off by default). Classes: 0 target verify
 * projection GEMMs (tcgen05), 1 target verify attention, 2 draft-model GEMMs, 3 draft
 * attention, 4 target LM-head GEMM (final + gated). Accumulated since the last reset:
 * total ms, launches, algorithmic bytes (weights + activations read + outputs written). */
faser_status faser_set_kernel_timing(faser_engine* e, int32_t enabled);
faser_status faser_kernel_stats(faser_engine* e, int32_t cls, double* ms, int64_t* launches,
                                double* bytes);
/* Algorithmic flops accumulated by the same timed launches (2 * N * K * rows for the GEMM
 * classes, 0 for attention): the tensor-pipe roofline basis when verify is TC-bound. */
faser_status faser_kernel_flops(faser_engine* e, int32_t cls, double* flops);

/* ABI self-description: FASER_ABI_VERSION and sizeof() of every struct above, in
 * declaration order (toy_params, exit_policy, gate_plan, gate_entry, overlap_plan,
 * latency_params, latency_model, verify_outcome, model_desc, engine_cfg, step_plan,
 * round_result, llama_shape, timeline_event, timeline_info). Writes min(n, 15) entries. */
int32_t faser_abi_version(void);
faser_status faser_abi_struct_sizes(int64_t* out, int32_t n);

/* ------------------------------------------------- host-side controllers (scalar math)
 * exitctl.cpp / overlap.cpp / latmodel.cpp restated natively; no device work. */

/* ExitPolicy::k_at (exitctl.cpp:9-17) for layer = 0..num_layers -> table[num_layers+1]. */
faser_status faser_k_table(const faser_exit_policy* policy, int32_t num_layers, int32_t* table);
/* LatencyModel::default_ground_truth (latmodel.cpp:396-403). */
void faser_default_latency_model(faser_latency_model* out);
/* eval_latency (latmodel.cpp:32-62); stage 0..3. */
faser_status faser_eval_latency(const faser_latency_model* m, int32_t stage, double b, double s,
                                double r, double* out_ms);
/* make_gate_plan (exitctl.cpp:70-82); models NULL = default ground truth. */
faser_status faser_make_gate_plan(const faser_exit_policy* policy, const faser_gate_entry* batch,
                                  int32_t n, double b, double r, const faser_latency_model* models,
                                  int32_t num_layers, faser_gate_plan* out);
/* plan_overlap (overlap.cpp:23-42). */
faser_status faser_plan_overlap(int32_t s, int32_t b, const faser_latency_model* models,
                                const double* r_grid, int32_t n_r, faser_overlap_plan* out);

/* --------------------------------------- per-request speculative-length controller (host)
 * AdaptiveDrafter / GpPosterior / AcceptanceBook / AcceptanceWindow (drafter.hpp:15-129,
 * drafter.cpp:14-230, sdcore.hpp:17-35) restated natively (the reference needs Eigen, which is
 * absent: parity of k_i assignment is unpinned). The GP posterior is computed from
 * per-candidate sufficient statistics (mathematically identical to the reference's LLT over
 * the raw window). */
typedef struct faser_drafter_cfg {
  int32_t n_candidates;
  int32_t candidates[16];      /* S = {1,2,3,4,5,6,8,10} (drafter.hpp:16) */
  int32_t window_ctx;          /* 64 */
  int32_t window_request;      /* 16 */
  int32_t reserved0;
  double epsilon;              /* 1e-6 */
  double kernel_len, kernel_var, noise_var; /* 1, 1, 0.1 */
  double cold_start_accept;    /* 0.7 */
} faser_drafter_cfg;

typedef struct faser_drafter faser_drafter;

void faser_drafter_default_cfg(faser_drafter_cfg* out);
faser_status faser_drafter_create(const faser_drafter_cfg* cfg, const faser_latency_model* models,
                                  faser_drafter** out);
void faser_drafter_destroy(faser_drafter* d);
/* Installs refreshed stage-latency models (the online profiler's periodic refit, PAPER.md:575
 * "refreshed every two hours in a separate process using runtime execution statistics"); the
 * GP windows and acceptance books are kept. */
faser_status faser_drafter_set_models(faser_drafter* d, const faser_latency_model* models);
/* AdaptiveDrafter::assign_lengths (drafter.cpp:175-207) for the batch (req_ids[n]), batch size
 * b and draft SM share r -> k_out[n]. */
faser_status faser_drafter_assign(faser_drafter* d, const int64_t* req_ids, int32_t n, int32_t b,
                                  double r, int32_t* k_out);
/* Feedback of one executed round: per request (spec, submitted, accepted) -> the request's
 * AcceptanceWindow (push, W = window_request) and the context AcceptanceBook; then
 * AdaptiveDrafter::observe_round(b, r, t_obs_ms, mean ratio per distinct spec length). */
faser_status faser_drafter_observe(faser_drafter* d, int32_t b, double r, double t_obs_ms,
                                   const int64_t* req_ids, const int32_t* spec,
                                   const int32_t* submitted, const int32_t* accepted, int32_t n);
/* Drops a finished request's acceptance window. */
faser_status faser_drafter_release(faser_drafter* d, int64_t req_id);
/* AcceptanceBook::estimate (drafter.cpp:151-161) for request req_ids[i] at length s[i] in the
 * (b, r) serving context: request window rate_for(s), else context rate, else context overall,
 * else request overall, else the cold-start default. Feeds the early-exit gate's GateEntry
 * accept_estimate (exitctl.hpp GateEntry, exitctl.cpp:19-46). */
faser_status faser_drafter_estimate(faser_drafter* d, const int64_t* req_ids, const int32_t* s, int32_t n,
                                    int32_t b, double r, double* a_hat);
/* The request's AcceptanceWindow (sdcore.cpp:8-35): out[j] = rate_for(qs[j]) for j < nq,
 * out[nq] = overall(); -1 when empty / unknown. */
faser_status faser_drafter_request_window(faser_drafter* d, int64_t req_id, const int32_t* qs, int32_t nq,
                                          double* out);
/* GpPosterior mu/sigma per candidate of context (b, r) and its round count (for tests). */
faser_status faser_drafter_posterior(faser_drafter* d, int32_t b, double r, double* mu,
                                     double* sigma, int32_t* rounds);
/* DrafterConfig::beta (drafter.cpp:14-17) and objective (drafter.cpp:19-23). */
double faser_drafter_beta(const faser_drafter_cfg* cfg, int32_t round);
faser_status faser_drafter_objective(double t_hat_ms, int32_t s, double a_hat, double epsilon,
                                     double* out);

/* Deterministic workload inputs (workload.cpp:116-122): synth_prompt. */
faser_status faser_synth_prompt(uint64_t seed, int32_t index, int32_t len, int32_t vocab,
                                int32_t* out);
/* Poisson arrivals over piecewise-constant rate segments (workload.cpp:73-98, synth_workload):
 * substreams "arrv" (exponential gaps) and "lens" (input then output length per record,
 * next_int modulo rule, rng.hpp:61-70). Writes min(n, cap) records, *n = total count. */
faser_status faser_synth_workload(const double* seg_duration_ms, const double* seg_rate_per_s,
                                  int32_t n_seg, int32_t in_lo, int32_t in_hi, int32_t out_lo,
                                  int32_t out_hi, uint64_t seed, double* arrival_ms,
                                  int32_t* in_len, int32_t* out_len, int32_t cap, int32_t* n);
/* Bursty sinusoidal rate profile (workload.cpp:100-114, sine_segments): `steps` segments of
 * duration_ms/steps at mean*(1 + a*sin(2*pi*(i+0.5)/steps)), a = (ptv-1)/(ptv+1). */
faser_status faser_sine_segments(double mean_rate_per_s, double peak_to_valley, double duration_ms,
                                 int32_t steps, double* seg_duration_ms, double* seg_rate_per_s);

#ifdef __cplusplus
}
#endif

#endif /* FASER_ENGINE_H */

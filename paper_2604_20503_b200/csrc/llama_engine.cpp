// llama_engine.cpp — host engine of the Llama-style speculative-decoding path (configs 3-5).
//
// Replaces the reference's SpeculativeEngine + Request loop (sdcore.hpp:39-116, driven by the
// missing serving loop SPEC.md:541-563) for transformer draft/target pairs:
//   submit()  -> pending queue; admitted at the next step (iteration-boundary admission,
//                B_max slots), prompt copied to HBM, both models prefilled (rows 0..len-2).
//   step()    -> ragged draft loop (step t runs the requests with min(k_i, remaining) > t,
//                one tcgen05 forward per step, sorted by k' so step t's rows are a prefix),
//                one verify forward over sum(k') rows with per-layer early-exit compaction,
//                fused accept + commit, ONE D2H of the round results, page release past the
//                committed length (KV rollback).
// Device memory: both models' weights (bf16), one page pool per model sharing one page table
// (draft and target cache the same positions), activations sized for max_batch x max_spec.
// Every failing CUDA call surfaces as FASER_ECUDA; there is no CPU fallback.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "faser/engine.h"
#include "llama.cuh"
#include "llama_engine.cuh"
#include "lanes.cuh"
#include "llama_step.cuh"
#include "tp.cuh"
#include "tc_gemm.cuh"
#include <nvtx3/nvToolsExt.h>

namespace faser {
namespace {

struct LFail {
  faser_status st;
  std::string msg;
};

#define LCK(call)                                                                         \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw LFail{FASER_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};      \
  } while (0)

struct Mem {
  void* p = nullptr;
  size_t bytes = 0;
  Mem() = default;
  Mem(const Mem&) = delete;
  Mem& operator=(const Mem&) = delete;
  ~Mem() {
    if (p) cudaFree(p);
  }
  void alloc(size_t b) {
    bytes = b;
    LCK(cudaMalloc(&p, b ? b : 16));
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

LlamaShape shape_of(const faser_llama_shape& s) {
  LlamaShape m{};
  m.d = s.d_model;
  m.layers = s.layers;
  m.n_q = s.n_heads;
  m.n_kv = s.n_kv_heads;
  m.hd = s.head_dim;
  m.ffn = s.ffn;
  m.vocab = s.vocab;
  m.rope_theta = static_cast<float>(s.rope_theta);
  m.eps = static_cast<float>(s.rms_eps);
  m.bigram_scale = static_cast<float>(s.bigram_scale);
  m.embed_noise = static_cast<float>(s.embed_noise);
  m.init_std = static_cast<float>(s.init_std);
  m.hard_fraction = s.hard_fraction;
  m.seed = s.seed;
  return m;
}

void validate_shape(const faser_llama_shape& s, const char* which) {
  auto bad = [&](const char* why) { throw LFail{FASER_EINVAL, std::string(which) + ": " + why}; };
  if (s.d_model <= 0 || s.d_model % 128) bad("d_model must be a positive multiple of 128");
  if (s.layers < 1 || s.layers > FASER_MAX_LAYERS) bad("layers out of range");
  if (s.head_dim != 64 && s.head_dim != 128) bad("head_dim must be 64 or 128");
  if (s.n_heads < 1 || s.n_kv_heads < 1 || s.n_heads % s.n_kv_heads) bad("n_heads must be a multiple of n_kv_heads");
  if ((s.n_heads / s.n_kv_heads) & (s.n_heads / s.n_kv_heads - 1)) bad("n_heads / n_kv_heads must be a power of two");
  if ((s.n_heads + 2 * s.n_kv_heads) * s.head_dim % 128) bad("qkv width must be a multiple of 128");
  if ((s.n_heads * s.head_dim) % 128) bad("n_heads*head_dim must be a multiple of 128");
  if (s.ffn <= 0 || s.ffn % 64) bad("ffn must be a positive multiple of 64");
  if (s.vocab < 2 || s.vocab % 128) bad("vocab must be a multiple of 128");
  if (!(s.rms_eps > 0) || !(s.rope_theta > 0) || !(s.init_std > 0)) bad("eps/theta/std must be > 0");
  if (!(s.hard_fraction >= 0.0 && s.hard_fraction <= 1.0)) bad("hard_fraction must lie in [0, 1]");
}

// ------------------------------------------------------------------ one model on device
struct LmModel {
  LlamaShape sh{};
  Mem arena;
  __nv_bfloat16* lm = nullptr;
  __nv_bfloat16* emb = nullptr;
  std::vector<LayerW> lw;
  GemmOperand op_lm;
  std::vector<GemmOperand> op_qkv, op_o, op_gu, op_d;
  Mem kv;
  int64_t kv_layer_stride = 0;
  Mem rope;  // float2 [max_pos][hd/2]

  int tp = 1, rank = 0;
  // `full` = the model's shape; with tp > 1 this rank holds the Megatron shard of the target:
  // n_q/tp query heads, n_kv/tp KV heads, ffn/tp FFN rows, vocab/tp LM-head rows (sh = local).
  void build(const LlamaShape& full, uint32_t ga, uint32_t gb, int n_pages, int max_pos, cudaStream_t st,
             int tp_ = 1, int rank_ = 0) {
    tp = tp_;
    rank = rank_;
    LlamaShape s = full;
    s.n_q /= tp;
    s.n_kv /= tp;
    s.ffn /= tp;
    // vocab-parallel LM head: ceil(V / tp) rows per rank rounded up to the 128-row tile; rank r
    // holds global ids [r * Vs, r * Vs + Vs), rows past V are zero padding masked out of the
    // argmax (EpiArgs::id_limit), so any V splits (config 5: 128256 over 8 ranks)
    if (tp > 1) s.vocab = ((full.vocab + tp - 1) / tp + 127) / 128 * 128;
    sh = s;
    const int64_t d = s.d, qkv = s.qkv_out(), qd = static_cast<int64_t>(s.n_q) * s.hd, F = s.ffn, V = s.vocab;
    const int64_t Vf = full.vocab, hd = s.hd;
    const int64_t per_layer = qkv * d + d * qd + 2 * F * d + d * F;
    const int64_t total = V * d + Vf * d + per_layer * s.layers;
    arena.alloc(total * 2);
    __nv_bfloat16* p = arena.as<__nv_bfloat16>();
    lm = p;
    emb = p + V * d;
    p += V * d + Vf * d;
    if (tp == 1) {
      LCK(lm_init_matrix(lm, V * d, s.seed, kTagLm * 4096u, s.init_std, st));
      LCK(lm_init_embedding(emb, lm, full, ga, gb, st));
    } else {  // the embedding needs the whole LM head (bigram construction); keep this rank's rows
      Mem full_lm;
      full_lm.alloc(static_cast<size_t>(Vf) * d * 2);
      LCK(lm_init_matrix(full_lm.as<__nv_bfloat16>(), Vf * d, s.seed, kTagLm * 4096u, s.init_std, st));
      LCK(lm_init_embedding(emb, full_lm.as<__nv_bfloat16>(), full, ga, gb, st));
      const int64_t valid = std::max<int64_t>(0, std::min<int64_t>(V, Vf - rank * V));  // rows < full vocab
      if (valid > 0)
        LCK(cudaMemcpyAsync(lm, full_lm.as<__nv_bfloat16>() + rank * V * d, valid * d * 2, cudaMemcpyDeviceToDevice, st));
      if (valid < V) LCK(cudaMemsetAsync(lm + valid * d, 0, (V - valid) * d * 2, st));
      LCK(cudaStreamSynchronize(st));
    }
    const int64_t nqf = full.n_q, nkvf = full.n_kv;
    for (int l = 0; l < s.layers; ++l) {
      LayerW w;
      __nv_bfloat16* wqkv = p;
      p += qkv * d;
      __nv_bfloat16* wo = p;
      p += d * qd;
      __nv_bfloat16* wgu = p;
      p += 2 * F * d;
      __nv_bfloat16* wd = p;
      p += d * F;
      const uint32_t tq = kTagQkv * 4096u + l;
      // column-parallel QKV: this rank's q rows, then its k rows, then its v rows
      LCK(lm_init_matrix(wqkv, s.n_q * hd * d, s.seed, tq, s.init_std, st, rank * s.n_q * hd * d));
      LCK(lm_init_matrix(wqkv + s.n_q * hd * d, s.n_kv * hd * d, s.seed, tq, s.init_std, st,
                         (nqf * hd + rank * s.n_kv * hd) * d));
      LCK(lm_init_matrix(wqkv + (s.n_q + s.n_kv) * hd * d, s.n_kv * hd * d, s.seed, tq, s.init_std, st,
                         (nqf * hd + nkvf * hd + rank * s.n_kv * hd) * d));
      // row-parallel O and down: this rank's input columns
      LCK(lm_init_cols(wo, d, nqf * hd, rank * qd, qd, s.seed, kTagO * 4096u + l, s.init_std, st));
      LCK(lm_init_gate_up(wgu, s.ffn, s.d, s.seed, l, s.init_std, st, static_cast<int64_t>(rank) * F));
      LCK(lm_init_cols(wd, d, static_cast<int64_t>(full.ffn), rank * F, F, s.seed, kTagDown * 4096u + l, s.init_std, st));
      w.wqkv = wqkv;
      w.wo = wo;
      w.wgu = wgu;
      w.wd = wd;
      lw.push_back(w);
      GemmOperand a, b, c, e;
      LCK(make_weight_operand(&a, wqkv, static_cast<int>(qkv), s.d));
      LCK(make_weight_operand(&b, wo, s.d, static_cast<int>(qd)));
      LCK(make_weight_operand(&c, wgu, 2 * s.ffn, s.d));
      LCK(make_weight_operand(&e, wd, s.d, s.ffn));
      op_qkv.push_back(a);
      op_o.push_back(b);
      op_gu.push_back(c);
      op_d.push_back(e);
    }
    LCK(make_weight_operand(&op_lm, lm, s.vocab, s.d));
    kv_layer_stride = static_cast<int64_t>(n_pages) * s.n_kv * 2 * kPage * s.hd;
    kv.alloc(static_cast<size_t>(kv_layer_stride) * s.layers * 2);
    LCK(cudaMemsetAsync(kv.p, 0, kv.bytes, st));  // stale pages must be finite (masked P*V)
    {  // TMA view of the pool for the attention kernel's page loads ([rows][hd], 64 x 64 boxes)
      const int64_t rows = kv_layer_stride * s.layers / s.hd;
      kv_tma = rows < (int64_t(1) << 31) && make_operand(&kv_op, kv.p, static_cast<int>(rows), s.hd, 64) == cudaSuccess;
    }
    // RoPE table (rotate-half), computed in double on the host; the oracle uses the same formula.
    const int half = s.hd / 2;
    std::vector<float> tab(static_cast<size_t>(max_pos) * half * 2);
    for (int pos = 0; pos < max_pos; ++pos)
      for (int i = 0; i < half; ++i) {
        const double inv = 1.0 / std::pow(static_cast<double>(s.rope_theta), (2.0 * i) / s.hd);
        const double a = pos * inv;
        tab[(static_cast<size_t>(pos) * half + i) * 2] = static_cast<float>(std::cos(a));
        tab[(static_cast<size_t>(pos) * half + i) * 2 + 1] = static_cast<float>(std::sin(a));
      }
    rope.alloc(tab.size() * 4);
    LCK(cudaMemcpyAsync(rope.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, st));
    LCK(cudaStreamSynchronize(st));  // tab is a host temporary
  }
  GemmOperand kv_op;
  bool kv_tma = false;
  KvDev kvdev(const int* ptab, int max_pages) const {
    KvDev k;
    k.pool = kv.as<__nv_bfloat16>();
    k.ptab = ptab;
    k.max_pages = max_pages;
    k.layer_stride = kv_layer_stride;
    k.tma = kv_tma ? &kv_op.map : nullptr;
    return k;
  }
};

// ------------------------------------------------------------------ activations of one model
struct LmWork {
  int rows_cap = 0, lm_rows_cap = 0;
  // residual stream: fp32 x, its bf16 copy xb (GEMM operand), per-128-column sums of squares
  Mem x, xb, ss, xs, xbs, sss;  // (+ scratch copies for early-exit compaction)
  Mem ob, q, h, logits, amax, attn, argmax, src_of;
  // fused exit-test estimator (target only): gathered W_lm[d] rows, z_d blocks [rows][128],
  // drafted id per row, per-(vocab tile, row) rank counts
  Mem wg, zd, row_d, rank_cnt;
  std::vector<GemmOperand> op_wg;  // one 128-row block of wg each
  size_t attn_bytes = 0;
  GemmOperand op_xb, op_ob, op_h;
  // persistent row metadata (draft steps)
  Mem meta;
  RowsDev rows{};

  void build(const LlamaShape& s, int cap, int lm_cap, bool rank = false) {
    rows_cap = cap;
    lm_rows_cap = lm_cap;
    const int64_t d = s.d, qd = static_cast<int64_t>(s.n_q) * s.hd;
    x.alloc(static_cast<size_t>(cap) * d * 4);
    xs.alloc(static_cast<size_t>(cap) * d * 4);
    xb.alloc(static_cast<size_t>(cap) * d * 2);
    xbs.alloc(static_cast<size_t>(cap) * d * 2);
    ss.alloc(static_cast<size_t>(cap) * (d / 128) * 4);
    sss.alloc(static_cast<size_t>(cap) * (d / 128) * 4);
    ob.alloc(static_cast<size_t>(cap) * qd * 2);
    q.alloc(static_cast<size_t>(cap) * qd * 2);
    h.alloc(static_cast<size_t>(cap) * s.ffn * 2);
    logits.alloc(static_cast<size_t>(lm_cap) * s.vocab * 4);
    amax.alloc(static_cast<size_t>(lm_cap) * (s.vocab / 128) * 8);
    attn_bytes = static_cast<size_t>(64) << 20;
    attn.alloc(attn_bytes);
    LCK(cudaMemset(attn.p, 0, size_t(1) << 20));  // split-KV counters (self-resetting)
    argmax.alloc(static_cast<size_t>(cap) * 4);
    src_of.alloc(static_cast<size_t>(cap) * 4);
    LCK(make_act_operand(&op_xb, xb.p, cap, s.d));
    LCK(make_act_operand(&op_ob, ob.p, cap, static_cast<int>(qd)));
    LCK(make_act_operand(&op_h, h.p, cap, s.ffn));
    if (rank) {
      const int blocks = (lm_cap + 127) / 128;
      wg.alloc(static_cast<size_t>(blocks) * 128 * d * 2);
      zd.alloc(static_cast<size_t>(blocks) * 128 * 128 * 4);
      row_d.alloc(static_cast<size_t>(blocks) * 128 * 4);
      rank_cnt.alloc(static_cast<size_t>(s.vocab / 128) * lm_cap * 4);
      op_wg.resize(blocks);
      for (int b = 0; b < blocks; ++b)
        LCK(make_weight_operand(&op_wg[b], wg.as<__nv_bfloat16>() + static_cast<size_t>(b) * 128 * d, 128, s.d));
    }
    meta.alloc(static_cast<size_t>(cap) * 9 * 4 + 64);
    int* m = meta.as<int>();
    rows.n_rows = m;
    m += 16;
    rows.row_req = m;
    m += cap;
    rows.row_pos = m;
    m += cap;
    rows.row_tok = m;
    m += cap;
    rows.row_j = m;
    m += cap;
    rows.req_first = m;
    m += cap;
    rows.req_n = m;
    m += cap;
    rows.req_slot = m;
    m += cap;
    rows.req_pos0 = m;
  }
};

// NVTX ranges of the step phases (host enqueue side; nsys / ncu --nvtx project them onto the
// GPU timeline). Header-only NVTX3: no cost unless a tool is attached.
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

int num_sms_dev() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

// ------------------------------------------------------------------ the engine
class LlamaEngine {
 public:
  faser_engine_cfg cfg{};
  faser_model_desc desc{};
  LlamaShape dsh{}, tsh{};
  LmModel draft, target;
  LmWork wd, wt;
  int tp = 1, tp_rank = 0;  // tensor-parallel verification of the target (tp.cuh)
  TpGroup* tpg = nullptr;
  Mem tp_part, tp_loc, tp_all;  // row-parallel partial [rows][d] bf16; argmax partials (float2)
  cudaStream_t stream = nullptr;   // draft lane (and everything in serial mode)
  cudaStream_t vstream = nullptr;  // verify lane of the overlapped (FULL) mode
  // admission-prefill lane (cfg.prefill_lane): newly admitted requests are prefilled on pstream
  // (lower priority, own work buffers) while the running batch drafts and verifies on `stream`;
  // they join the batch at the next step, whose start waits for the prefill
  cudaStream_t pstream = nullptr;
  // In-flight prefill batches, oldest first: the requests they prefill stay out of the steps
  // until their event completes (polled at each step start, never waited on while other
  // requests can run). Each batch's row metadata lives in its own step blob, so the blobs form a
  // ring of kBlobs and a blob is reused only once no in-flight batch reads it.
  struct PfBatch {
    int blob;
    std::vector<int64_t> ids;
  };
  std::deque<PfBatch> pf_q;
  cudaEvent_t ev_pf_go = nullptr;
  static constexpr int kBlobs = 16;  // > the prefill batches in flight at B = 256 (admission bursts)
  cudaEvent_t ev_pf_done[kBlobs] = {};  // per blob
  bool pf_lane = false;
  int skip_mask = -1;  // faser_debug_set_skip_mask (timing experiments); -1: FASER_SKIP
  float samp_inv_tau = 0.f;  // faser_set_sampling: > 0 = coupled Gumbel-max sampling at 1 / tau
  uint64_t samp_seed = 0;
  bool pf_defer = false;  // this step: new requests wait for the lane to drain
  int pf_in_flight_cap = 2;  // FASER_PF_INFLIGHT
  double pf_wait_ms = 0.0;  // host time blocked on a prefill (nothing runnable / blob ring full)
  int64_t pf_waits = 0;
  LmWork wd_pf, wt_pf;
  std::vector<int64_t> run;  // the requests this step drafts and verifies
  cudaStream_t fs = nullptr;       // stream the current forward() launches on
  cudaEvent_t ev[4] = {};
  cudaEvent_t ev_chunk[FASER_MAX_SPEC + 1] = {};
  // overlapped mode: SM-partitioned lanes and the measured pipeline timeline of the last step
  std::unique_ptr<SmLanes> lanes;
  int fwd_sms = 148;  // SM count the current forward's GEMM plans size their grids for
  static constexpr int kLaneRec = 2 * (FASER_MAX_SPEC + 2), kLaneDec = FASER_MAX_SPEC + 2;
  static constexpr int kLaneRes = FASER_MAX_SPEC + 2;
  static constexpr int kLaneInts = kLaneRec + kLaneDec + kLaneRes + 2;
  cudaEvent_t ev_fork = nullptr, ev_dend = nullptr;
  cudaEvent_t ev_d0[FASER_MAX_SPEC + 1] = {}, ev_d1[FASER_MAX_SPEC + 1] = {};
  cudaEvent_t ev_v0[FASER_MAX_SPEC + 1] = {}, ev_v1[FASER_MAX_SPEC + 1] = {};
  int32_t* h_lane = nullptr;
  bool tl_valid = false;
  int tl_nch = 0, tl_lane_mode = 0;
  LanePair tl_lp;
  std::vector<faser_timeline_event> tl_events;
  faser_timeline_info tl_info{};
  int nsm = 148;
  bool graph_mode = false;  // FASER_CUDA_GRAPH=1: each step is captured and replayed as one graph
  int max_spec = 16;
  int max_seq = 0;    // slot row capacity (tokens)
  int max_pages = 0;  // pages per slot
  int n_pages = 0;
  int eos = 0;
  std::string err;
  int64_t launches = 0, h2d = 0, d2h = 0;
  float t_draft = 0.f, t_verify = 0.f, t_step = 0.f, t_prefill = 0.f;

  // slots
  Mem s_tok, s_len, s_ncomm, s_maxout, s_done, s_exempt, ptab;
  LmSlots sl{};
  // per-request step state (sorted order), persistent
  Mem r_drafted, r_count, r_active, r_gl, r_npl, r_pl, r_prl, r_pr, r_fail, r_truth, r_truth_rj, r_span;
  LmReqState rq{};
  LmReqState cur_q{};  // rq + this step's per-request arrays (slot, k, ...) in the blob
  // step blob
  Mem d_blobs[kBlobs];
  char* h_blobs[kBlobs] = {};
  int blob_i = 0;
  char* h_blob = nullptr;  // the current step's blob (host, pinned) and its device copy
  char* d_blob = nullptr;
  size_t blob_cap = 0;
  faser_round_result* h_res = nullptr;
  Mem d_res;

  struct Req {
    int64_t id;
    std::vector<int32_t> prompt, committed;
    int32_t max_out = 0, spec = 0, slot = -1, len = 0;
    bool done = false, admitted = false;
    bool prefilling = false;  // admission prefill in flight on the prefill lane
    std::vector<int32_t> pages;
  };
  std::unordered_map<int64_t, Req> reqs;
  std::deque<int64_t> pending;
  std::vector<int64_t> live;
  std::vector<int32_t> free_slots;
  std::set<int32_t> free_pages;  // deterministic: lowest page id first

  // debug capture
  struct Stage {
    int rows = 0;
    std::vector<float> logits;
    std::vector<int64_t> ids;
  };
  std::map<int, Stage> stages;
  std::vector<int32_t> dbg_drafted;  // live order [n][MAX_SPEC]
  std::vector<int64_t> step_sorted_ids;

  ~LlamaEngine() {
    if (stream) cudaStreamSynchronize(stream);
    if (getenv("FASER_PF_DEBUG") && pstream)
      fprintf(stderr, "prefill lane: %lld host waits, %.2f ms blocked; host step %.1f ms (main enqueue %.1f, prefill enqueue %.1f, sync %.1f)\n",
              static_cast<long long>(pf_waits), pf_wait_ms, h_step_ms, h_main_ms, h_pfenq_ms, h_sync_ms);
    for (auto& kv : reqs) (void)kv;
    for (char* hb : h_blobs)
      if (hb) cudaFreeHost(hb);
    if (h_res) cudaFreeHost(h_res);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : ev_chunk)
      if (e) cudaEventDestroy(e);
    for (auto* arr : {ev_d0, ev_d1, ev_v0, ev_v1})
      for (int i = 0; i <= FASER_MAX_SPEC; ++i)
        if (arr[i]) cudaEventDestroy(arr[i]);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_dend) cudaEventDestroy(ev_dend);
    if (h_lane) cudaFreeHost(h_lane);
    lanes.reset();
    if (vstream) cudaStreamDestroy(vstream);
    if (pstream) {
      cudaStreamSynchronize(pstream);
      cudaStreamDestroy(pstream);
    }
    if (ev_pf_go) cudaEventDestroy(ev_pf_go);
    for (auto e : ev_pf_done)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }

  void create(const faser_model_desc* m, const faser_engine_cfg* c) {
    cfg = *c;
    desc = *m;
    validate_shape(m->draft, "draft");
    validate_shape(m->target, "target");
    if (m->draft.vocab != m->target.vocab) throw LFail{FASER_EINVAL, "draft and target vocab differ"};
    if (cfg.max_batch < 1 || cfg.max_batch > 1024) throw LFail{FASER_EINVAL, "max_batch out of range [1, 1024]"};
    if (cfg.max_seq_len < 2) throw LFail{FASER_EINVAL, "max_seq_len must be >= 2"};
    if (cfg.mode < FASER_MODE_VSD || cfg.mode > FASER_MODE_FULL) throw LFail{FASER_EINVAL, "unknown mode"};
    if (cfg.exempt_rule < 0 || cfg.exempt_rule > 2) throw LFail{FASER_EINVAL, "exempt_rule must be 0, 1 or 2"};
    if (cfg.exempt_rule == 2 && cfg.mode == FASER_MODE_FULL)
      throw LFail{FASER_EINVAL, "recovery on prune (exempt_rule 2) is a serial-verify mode; not with FULL"};
    const faser_exit_policy& p = cfg.exit_policy;
    if (p.k_init < 1 || p.k_final < 1 || p.k_final > p.k_init)
      throw LFail{FASER_EINVAL, "exit policy thresholds must satisfy k_init >= k_final >= 1"};
    max_spec = cfg.max_spec_length > 0 ? cfg.max_spec_length : 16;
    if (max_spec > FASER_MAX_SPEC) throw LFail{FASER_EINVAL, "max_spec_length > FASER_MAX_SPEC"};
    if (cfg.default_spec_length < 1 || cfg.default_spec_length > max_spec)
      throw LFail{FASER_EINVAL, "default_spec_length out of range"};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw LFail{FASER_ECUDA, "no CUDA device available"};
    if (cfg.device < 0 || cfg.device >= ndev) throw LFail{FASER_EINVAL, "device index out of range"};
    LCK(cudaSetDevice(cfg.device));
    nsm = num_sms_dev();
    graph_mode = getenv("FASER_CUDA_GRAPH") && getenv("FASER_CUDA_GRAPH")[0] == '1';
    dsh = shape_of(m->draft);
    tsh = shape_of(m->target);
    eos = tsh.vocab - 1;
    LCK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    {
      // verify lane priority (FASER_VERIFY_PRIO: 0 = same as the draft lane, 1 = verify first,
      // 2 = draft first): decides whose CTAs the scheduler dispatches first when the two
      // overlapped lanes both have work queued
      int lo = 0, hi = 0;
      LCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const int mode = getenv("FASER_VERIFY_PRIO") ? atoi(getenv("FASER_VERIFY_PRIO")) : 0;
      if (mode == 2) {
        LCK(cudaStreamDestroy(stream));
        LCK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, hi));
        fs = stream;
      }
      LCK(cudaStreamCreateWithPriority(&vstream, cudaStreamNonBlocking, mode == 1 ? hi : lo));
    }
    fs = stream;
    pf_lane = cfg.prefill_lane != 0 && !(cfg.tp_size > 1) && cfg.mode != FASER_MODE_FULL && !graph_mode;
    if (pf_lane) {
      // the running batch's stream gets the higher priority: prefill CTAs fill the SMs its
      // latency-bound draft / verify kernels leave idle
      int lo = 0, hi = 0;
      LCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      LCK(cudaStreamDestroy(stream));
      LCK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, hi));
      fs = stream;
      LCK(cudaStreamCreateWithPriority(&pstream, cudaStreamNonBlocking, lo));
      if (getenv("FASER_PF_INFLIGHT")) pf_in_flight_cap = std::max(1, atoi(getenv("FASER_PF_INFLIGHT")));
      LCK(cudaEventCreateWithFlags(&ev_pf_go, cudaEventDisableTiming));
      for (auto& e : ev_pf_done) LCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (auto& e : ev) LCK(cudaEventCreate(&e));
    for (auto& e : ev_chunk) LCK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto* arr : {ev_d0, ev_d1, ev_v0, ev_v1})
      for (int i = 0; i <= FASER_MAX_SPEC; ++i) LCK(cudaEventCreate(&arr[i]));
    LCK(cudaEventCreate(&ev_fork));
    LCK(cudaEventCreateWithFlags(&ev_dend, cudaEventDisableTiming));
    LCK(cudaMallocHost(reinterpret_cast<void**>(&h_lane), sizeof(int32_t) * kLaneInts));
    fwd_sms = nsm;
    max_seq = cfg.max_seq_len + max_spec + 2;
    max_pages = (max_seq + kPage - 1) / kPage;
    n_pages = cfg.max_batch * max_pages;
    const int B = cfg.max_batch;
    const int prefill_rows = cfg.prefill_rows > 0 ? cfg.prefill_rows : 8192;
    const int verify_rows = B * max_spec;
    const int cap = std::max({prefill_rows, verify_rows, cfg.max_seq_len});
    tp = cfg.tp_size > 1 ? cfg.tp_size : 1;
    tp_rank = tp > 1 ? cfg.tp_rank : 0;
    if (tp > 1) {
      tpg = tp_group_of(cfg.tp_group);
      if (!tpg || tpg->size != tp) throw LFail{FASER_EINVAL, "tp_group missing or of a different size"};
      if (tp_rank < 0 || tp_rank >= tp) throw LFail{FASER_EINVAL, "tp_rank out of range"};
      if (cfg.mode != FASER_MODE_VSD && cfg.mode != FASER_MODE_VSD_AD)
        throw LFail{FASER_EINVAL, "tensor-parallel verification supports modes VSD and VSD_AD"};
      if (cfg.debug_capture) throw LFail{FASER_EINVAL, "debug_capture is not available with tp_size > 1"};
      const faser_llama_shape& t = m->target;
      if (t.n_heads % tp || t.n_kv_heads % tp || t.ffn % (64 * tp) ||
          ((t.n_heads + 2 * t.n_kv_heads) / tp * t.head_dim) % 128 || (t.n_heads / tp * t.head_dim) % 128)
        throw LFail{FASER_EINVAL, "target shape does not split over tp_size ranks"};
    }
    draft.build(dsh, m->bigram_a, m->bigram_b, n_pages, max_seq, stream);
    target.build(tsh, m->bigram_a, m->bigram_b, n_pages, max_seq, stream, tp, tp_rank);
    wd.build(dsh, cap, B);
    wt.build(target.sh, cap, verify_rows, cfg.mode >= FASER_MODE_VSD_AD_EE);
    if (pf_lane) {  // the prefill lane's own activations (no logits: lm rows 1)
      const int pcap = std::max(prefill_rows, cfg.max_seq_len);
      wd_pf.build(dsh, pcap, 1);
      wt_pf.build(target.sh, pcap, 1);
    }
    if (tp > 1) {
      tp_part.alloc(static_cast<size_t>(cap) * tsh.d * 2);
      tp_loc.alloc(static_cast<size_t>(cap) * 8);
      tp_all.alloc(static_cast<size_t>(cap) * 8 * tp);
    }
    LCK(cudaDeviceSynchronize());
    s_tok.alloc(static_cast<size_t>(B) * max_seq * 4);
    s_len.alloc(B * 4);
    s_ncomm.alloc(B * 4);
    s_maxout.alloc(B * 4);
    s_done.alloc(B * 4);
    s_exempt.alloc(B * 4);
    ptab.alloc(static_cast<size_t>(B) * max_pages * 4);
    LCK(cudaMemsetAsync(ptab.p, 0, ptab.bytes, stream));
    sl.tok = s_tok.as<int32_t>();
    sl.len = s_len.as<int32_t>();
    sl.ncomm = s_ncomm.as<int32_t>();
    sl.max_out = s_maxout.as<int32_t>();
    sl.done = s_done.as<int32_t>();
    sl.exempt = s_exempt.as<int32_t>();
    sl.max_seq = max_seq;
    r_drafted.alloc(static_cast<size_t>(B) * FASER_MAX_SPEC * 4);
    r_count.alloc(B * 4);
    r_active.alloc(B * 4);
    r_gl.alloc(B * 4);
    r_npl.alloc(B * 4);
    r_pl.alloc(static_cast<size_t>(B) * FASER_MAX_SPEC * 4);
    r_prl.alloc(static_cast<size_t>(B) * FASER_MAX_SPEC * 4);
    r_pr.alloc(B * 8);
    r_fail.alloc(B * 4);
    r_truth.alloc(static_cast<size_t>(cap) * 4);
    r_truth_rj.alloc(static_cast<size_t>(B) * FASER_MAX_SPEC * 4);
    r_span.alloc(B * 4);
    rq.drafted = r_drafted.as<int32_t>();
    rq.count = r_count.as<int32_t>();
    rq.active = r_active.as<int32_t>();
    rq.gate_layers = r_gl.as<int32_t>();
    rq.n_pl = r_npl.as<int32_t>();
    rq.pl = r_pl.as<int32_t>();
    rq.prune_layer = r_prl.as<int32_t>();
    rq.pr = r_pr.as<int32_t>();
    rq.failmask = r_fail.as<uint32_t>();
    rq.truth = r_truth.as<int32_t>();
    rq.truth_rj = r_truth_rj.as<int32_t>();
    rq.span = r_span.as<int32_t>();
    // blob: request arrays (5n) + verify rows (4T + 4n + 16) + ptab triples + admits + prefill rows
    blob_cap = static_cast<size_t>(B) * 64 + static_cast<size_t>(verify_rows) * 16 +
               static_cast<size_t>(B) * max_pages * 12 + static_cast<size_t>(B) * sizeof(LmAdmit) +
               static_cast<size_t>(cap) * 16 + static_cast<size_t>(B) * 16 * 2 + 4096 +
               static_cast<size_t>(B) * cfg.max_seq_len * (4 + 16) +   // prompts + prefill rows
               static_cast<size_t>(B) * (9 * 4 + 64) +                  // per-chunk arrays
               sizeof(int32_t) * kLaneInts + 64;                        // lane state
    for (int b = 0; b < (pf_lane ? kBlobs : 1); ++b) {
      LCK(cudaMallocHost(reinterpret_cast<void**>(&h_blobs[b]), blob_cap));
      d_blobs[b].alloc(blob_cap);
    }
    h_blob = h_blobs[0];
    d_blob = d_blobs[0].as<char>();
    LCK(cudaMallocHost(reinterpret_cast<void**>(&h_res), sizeof(faser_round_result) * B));
    d_res.alloc(sizeof(faser_round_result) * B);
    for (int s = B - 1; s >= 0; --s) free_slots.push_back(s);
    for (int p = 0; p < n_pages; ++p) free_pages.insert(p);
    LCK(cudaStreamSynchronize(stream));
  }

  // ---------------------------------------------------------------- forward
  struct VChunk {
    RowsDev rows;
    int T = 0, max_rows = 0;
  };
  bool use_graph_mode() const { return graph_mode && cfg.debug_capture == 0; }
  struct Fwd {
    RowsDev rows;
    int T = 0, n_req = 0, max_rows = 0, max_ctx = 0;
    bool logits = false;
    int* argmax_out = nullptr;
    bool ee = false;
    int gate_lo = 0, gate_hi = 0;
    const int* k_table = nullptr;
    bool capture = false;
    int64_t kv_tokens = 0;  // sum over requests of the context each attention call reads
    bool pre_embedded = false;  // rows' embeddings already written (fused draft control kernel)
    bool skip_argmax = false;   // leave the LM head's per-tile (max, id) partials for the caller
    int q0 = 0;                 // first drafted position of the rows (overlapped chunk start)
  };

  GemmPlan plan(int n_out, int T, int k) const { return gemm_plan(n_out, T, k, fwd_sms); }
  // ---- per-kernel-class timing (opt-in): event pairs around launches, resolved after the step
  static constexpr int kClasses = 5;
  bool ktiming = false;
  struct KPend {
    int cls;
    cudaEvent_t a, b;
    double bytes, flops;
    int n;  // launches between the event pair (a run of back-to-back same-class launches)
  };
  std::vector<KPend> kpend;
  std::vector<cudaEvent_t> kpool;
  double k_ms[kClasses] = {}, k_bytes[kClasses] = {}, k_flops[kClasses] = {};
  int64_t k_n[kClasses] = {};
  cudaEvent_t kev() {
    if (kpool.empty()) {
      cudaEvent_t e;
      LCK(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = kpool.back();
    kpool.pop_back();
    return e;
  }
  // `n` > 1: `launch` enqueues a run of n back-to-back launches of the class; one event pair
  // brackets the run, so the programmatic (PDL) overlap between them stays intact (an event
  // record between two launches serialises them) and the run's time is split evenly.
  template <class F>
  void timed(int cls, double bytes, F&& launch, double flops = 0.0, int n = 1) {
    if (!ktiming || capturing || cls < 0) {
      launch();
      return;
    }
    KPend p{cls, kev(), kev(), bytes, flops, n};
    LCK(cudaEventRecord(p.a, fs));
    launch();
    LCK(cudaEventRecord(p.b, fs));
    kpend.push_back(p);
  }
  void resolve_kernel_timing() {
    for (KPend& p : kpend) {
      float ms = 0.f;
      LCK(cudaEventSynchronize(p.b));
      LCK(cudaEventElapsedTime(&ms, p.a, p.b));
      k_ms[p.cls] += ms;
      k_bytes[p.cls] += p.bytes;
      k_flops[p.cls] += p.flops;
      k_n[p.cls] += p.n;
      kpool.push_back(p.a);
      kpool.push_back(p.b);
    }
    kpend.clear();
  }
  bool capturing = false;
  cudaError_t record_event(cudaEvent_t e) {
    return capturing ? cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal) : cudaEventRecord(e, stream);
  }

  void capture_stage(int stage, const LmModel& m, const LmWork& w, const Fwd& f) {
    LCK(cudaStreamSynchronize(fs));
    int n = 0;
    LCK(cudaMemcpy(&n, f.rows.n_rows, 4, cudaMemcpyDeviceToHost));
    const int V = m.sh.vocab;
    Stage st;
    st.rows = n;
    st.logits.resize(static_cast<size_t>(n) * V);
    LCK(cudaMemcpy(st.logits.data(), w.logits.p, st.logits.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<int> req(n), jj(n);
    LCK(cudaMemcpy(req.data(), f.rows.row_req, 4 * n, cudaMemcpyDeviceToHost));
    LCK(cudaMemcpy(jj.data(), f.rows.row_j, 4 * n, cudaMemcpyDeviceToHost));
    st.ids.resize(2 * static_cast<size_t>(n));
    for (int r = 0; r < n; ++r) {
      st.ids[2 * r] = step_sorted_ids[req[r]];
      st.ids[2 * r + 1] = jj[r];
    }
    stages[stage] = std::move(st);
  }

  void forward(LmModel& m, LmWork& w, const Fwd& f) {
    const LlamaShape& s = m.sh;
    const int T = f.T;
    if (T <= 0) return;
    if (T > w.rows_cap) throw LFail{FASER_ECAPACITY, "forward rows exceed capacity"};
    const bool lm_head = f.logits || f.ee;
    if (lm_head && T > w.lm_rows_cap) throw LFail{FASER_ECAPACITY, "LM-head rows exceed capacity"};
    const KvDev kv = m.kvdev(ptab.as<int>(), max_pages);
    const int qd = s.n_q * s.hd;
    // prefill forwards (no logits) take the prefill plan
    auto pl = [&](int n_out, int k) { return f.logits ? plan(n_out, T, k) : gemm_plan_prefill(n_out, T, k, fwd_sms); };
    const GemmPlan p_qkv = pl(s.qkv_out(), s.d), p_o = pl(s.d, qd);
    const GemmPlan p_gu = pl(2 * s.ffn, s.d), p_d = pl(s.d, s.ffn), p_lm = plan(s.vocab, T, s.d);
    RowsDev rows = f.rows;
    EpiArgs base;
    base.t_stride = T;
    base.n_rows = rows.n_rows;
    base.ss_chunks = s.d / 128;
    base.d_norm = s.d;
    base.eps = s.eps;
    EpiArgs e_qkv = base;
    e_qkv.mode = kEpiQkv;
    e_qkv.ss_in = w.ss.as<float>();
    e_qkv.rows = rows;
    e_qkv.rope = m.rope.as<float2>();
    e_qkv.kv = kv;
    e_qkv.n_q = s.n_q;
    e_qkv.n_kv = s.n_kv;
    e_qkv.hd = s.hd;
    e_qkv.q = w.q.as<__nv_bfloat16>();
    EpiArgs e_res = base;
    e_res.mode = kEpiResid;
    e_res.x = w.x.as<float>();
    e_res.xb = w.xb.as<__nv_bfloat16>();
    e_res.ss_out = w.ss.as<float>();
    EpiArgs e_glu = base;
    e_glu.mode = kEpiSwiglu;
    e_glu.ss_in = w.ss.as<float>();
    e_glu.h = w.h.as<__nv_bfloat16>();
    e_glu.ffn = s.ffn;
    const bool is_tp_target = tp > 1 && &m == &target;
    EpiArgs e_part = base;  // row-parallel TP partial (bf16 [T][d], summed over ranks afterwards)
    e_part.mode = kEpiStore;
    e_part.out_bf16 = tp_part.as<__nv_bfloat16>();
    EpiArgs e_lm = base;
    if (is_tp_target) {
      e_lm.id_off = tp_rank * s.vocab;  // global token ids of this vocab shard
      e_lm.id_limit = tsh.vocab;        // padding rows of the last shard(s) never win the argmax
    }
    e_lm.mode = kEpiLogits;
    e_lm.ss_in = w.ss.as<float>();
    e_lm.logits = w.logits.as<float>();
    e_lm.amax = w.amax.as<float2>();
    if (samp_inv_tau > 0.f && f.logits) {  // draft steps and verify: sample, keyed by (request, position)
      e_lm.rows = rows;
      e_lm.req_ids = cur_q.req_id;
      e_lm.samp_seed = samp_seed;
      e_lm.inv_tau = samp_inv_tau;
    }

    if (!f.pre_embedded) {
      LCK(lm_embed(s, m.emb, rows, T, w.x.as<float>(), w.xb.as<__nv_bfloat16>(), w.ss.as<float>(), fs));
      ++launches;
    }
    // kernel classes for timing: target verify (logits) vs draft model; prefill untimed
    const bool is_target = &m == &target;
    const int gcls = f.logits ? (is_target ? 0 : 2) : -1;
    const int acls = f.logits ? (is_target ? 1 : 3) : -1;
    // algorithmic bytes of one projection launch: weights + activation rows in (bf16) + out
    auto gbytes = [&](int64_t n_out, int64_t k, int64_t out_cols) {
      return 2.0 * n_out * k + 2.0 * T * k + 2.0 * T * out_cols;
    };
    auto gflops = [&](int64_t n_out, int64_t k) { return 2.0 * n_out * k * T; };
    // attention: the K/V bytes every request reads (its context incl. the new rows) + q/o
    const double abytes = static_cast<double>(f.kv_tokens) * 2 * s.n_kv * s.hd * 2 + 4.0 * T * s.n_q * s.hd;
    // timing experiments only (FASER_SKIP bitmask, target verify forward): 1 attention, 2 qkv,
    // 4 o, 8 gate/up, 16 down — results are garbage, the step time shows each class's share
    static const int skip_env0 = getenv("FASER_SKIP") ? atoi(getenv("FASER_SKIP")) : 0;
    const int skip_env = skip_mask >= 0 ? skip_mask : skip_env0;
    // (bit 32: apply the mask to prefill forwards of both models instead)
    const int skip = (skip_env & 32) ? (!f.logits ? (skip_env & 31) : 0) : ((f.logits && is_target) ? skip_env : 0);
    for (int l = 0; l < s.layers; ++l) {
      e_qkv.layer = l;
      if (!(skip & 2))
      timed(gcls, gbytes(s.qkv_out(), s.d, s.qkv_out()),
            [&] { LCK(gemm_fused(m.op_qkv[l], w.op_xb, T, p_qkv, e_qkv, fs)); }, gflops(s.qkv_out(), s.d));
      if (!(skip & 1))
      timed(acls, abytes, [&] {
        LCK(lm_attention(s, rows, f.n_req, f.max_rows, f.max_ctx, kv, l, w.q.as<__nv_bfloat16>(),
                         w.ob.as<__nv_bfloat16>(), w.attn.as<float>(), w.attn_bytes, fs));
      });
      const bool tp_rows = is_tp_target;  // row-parallel: partial sums -> all-reduce -> residual add
      auto row_parallel = [&](const GemmOperand& wop, const GemmOperand& xop, const GemmPlan& pl) {
        LCK(gemm_fused(wop, xop, T, pl, e_part, fs));
        LCK(tpg->allreduce_sum(tp_rank, tp_part.as<__nv_bfloat16>(), static_cast<size_t>(T) * s.d, fs));
        LCK(tp_resid_add(tp_part.as<__nv_bfloat16>(), w.x.as<float>(), w.xb.as<__nv_bfloat16>(), w.ss.as<float>(), T, s.d, fs));
        launches += 2;
      };
      if (!tp_rows && !(skip & 28)) {
        // o -> gate/up -> down run back to back: one event pair around the run
        timed(gcls, gbytes(s.d, qd, s.d) + gbytes(2 * s.ffn, s.d, s.ffn) + gbytes(s.d, s.ffn, s.d), [&] {
          LCK(gemm_fused(m.op_o[l], w.op_ob, T, p_o, e_res, fs));
          LCK(gemm_fused(m.op_gu[l], w.op_xb, T, p_gu, e_glu, fs));
          LCK(gemm_fused(m.op_d[l], w.op_h, T, p_d, e_res, fs));
        }, gflops(s.d, qd) + gflops(2 * s.ffn, s.d) + gflops(s.d, s.ffn), 3);
      } else {
        if (tp_rows)
          row_parallel(m.op_o[l], w.op_ob, p_o);
        else if (!(skip & 4))
          timed(gcls, gbytes(s.d, qd, s.d), [&] { LCK(gemm_fused(m.op_o[l], w.op_ob, T, p_o, e_res, fs)); },
                gflops(s.d, qd));
        if (!(skip & 8))
        timed(gcls, gbytes(2 * s.ffn, s.d, s.ffn), [&] { LCK(gemm_fused(m.op_gu[l], w.op_xb, T, p_gu, e_glu, fs)); },
              gflops(2 * s.ffn, s.d));
        if (tp_rows)
          row_parallel(m.op_d[l], w.op_h, p_d);
        else if (!(skip & 16))
          timed(gcls, gbytes(s.d, s.ffn, s.d), [&] { LCK(gemm_fused(m.op_d[l], w.op_h, T, p_d, e_res, fs)); },
                gflops(s.d, s.ffn));
      }
      launches += 5;
      const int layer = l + 1;  // residual now holds the output of `layer` layers
      if (f.ee && layer >= f.gate_lo && layer < f.gate_hi && layer < s.layers) {
        // fused exit-test estimator (no top-K, no T x V logits): z_d of every
        // row through the LM head's own accumulation order (W_lm[d] gathered, one 128 x 128
        // block-diagonal launch per 128 rows), then the LM head counts the outranking ids per
        // tile in its epilogue and exit_rank sums them
        LCK(lm_rank_prep(cur_q, rows, m.lm, s.d, w.wg.as<__nv_bfloat16>(), w.row_d.as<int>(), T, fs));
        GemmPlan pz;
        pz.bn = 128;
        pz.mc = 1;
        pz.splits = 1;  // K order of the LM head (splits = 1)
        pz.deep = true;
        for (int b = 0; b * 128 < T; ++b) {
          EpiArgs ez = base;
          ez.mode = kEpiStore;
          ez.ss_in = w.ss.as<float>();
          ez.out = w.zd.as<float>();
          ez.t_begin = b * 128;
          ez.w_after_wait = 1;  // wg was written by rank_prep: no weight prefetch before the PDL wait
          LCK(gemm_fused(w.op_wg[b], w.op_xb, 128, pz, ez, fs));
        }
        EpiArgs e_rank = e_lm;
        e_rank.mode = kEpiRank;
        e_rank.logits = f.capture ? w.logits.as<float>() : nullptr;
        e_rank.amax = nullptr;
        e_rank.zd_src = w.zd.as<float>();
        e_rank.row_d = w.row_d.as<int>();
        e_rank.rank_cnt = w.rank_cnt.as<int>();
        LCK(gemm_fused(m.op_lm, w.op_xb, T, p_lm, e_rank, fs));
        if (f.capture) capture_stage(layer, m, w, f);
        LCK(lm_exit_rank(sl, cur_q, rows, w.rank_cnt.as<int>(), s.vocab / 128, T, f.k_table[layer], T, fs));
        launches += 3 + (T + 127) / 128;
        LCK(lm_frontier_compact(sl, cur_q, rows, f.n_req, layer, w.src_of.as<int>(), fs, f.q0,
                                cfg.exempt_rule == 2 ? 1 : 0, s.layers));
        LCK(lm_gather_rows(rows, w.src_of.as<int>(), s.d, T, w.x.as<float>(), w.xb.as<__nv_bfloat16>(),
                           w.ss.as<float>(), w.xs.as<float>(), w.xbs.as<__nv_bfloat16>(), w.sss.as<float>(),
                           fs));
        launches += 2;
      }
    }
    if (f.logits) {
      // the final head needs only the per-tile (max, id) partials; the T x V logits are written
      // for validation (debug capture) only
      EpiArgs e_fin = e_lm;
      if (!f.capture) e_fin.logits = nullptr;
      timed(is_target ? 4 : 2, gbytes(s.vocab, s.d, f.capture ? 2 * s.vocab : 0),
            [&] { LCK(gemm_fused(m.op_lm, w.op_xb, T, p_lm, e_fin, fs)); }, gflops(s.vocab, s.d));
      if (is_tp_target) {  // vocab-parallel greedy argmax: all-gather (max, lowest global id) per row
        LCK(tp_local_argmax(s.vocab / 128, T, w.amax.as<float2>(), tp_loc.as<float2>(), fs));
        LCK(tpg->allgather_f2(tp_rank, tp_loc.as<float2>(), tp_all.as<float2>(), static_cast<size_t>(T), fs));
        LCK(tp_merge_argmax(tp, T, tp_all.as<float2>(), f.argmax_out, fs));
        launches += 2;
      } else if (!f.skip_argmax) {
        LCK(lm_argmax_reduce(s.vocab / 128, rows, T, w.amax.as<float2>(), f.argmax_out, fs));
      }
      launches += 2;
      if (f.capture) capture_stage(0, m, w, f);
    }
  }

  // ---------------------------------------------------------------- pages
  void ensure_pages(Req& r, int upto_pos) {  // positions [0, upto_pos] backed
    const int need = upto_pos / kPage + 1;
    if (need > max_pages) throw LFail{FASER_ECAPACITY, "sequence exceeds page capacity"};
    while (static_cast<int>(r.pages.size()) < need) {
      if (free_pages.empty()) throw LFail{FASER_ENOMEM, "KV page pool exhausted"};
      const int p = *free_pages.begin();
      free_pages.erase(free_pages.begin());
      pend_triples.push_back(r.slot);
      pend_triples.push_back(static_cast<int>(r.pages.size()));
      pend_triples.push_back(p);
      r.pages.push_back(p);
    }
  }
  void release_pages_beyond(Req& r, int keep_pages) {
    while (static_cast<int>(r.pages.size()) > keep_pages) {
      free_pages.insert(r.pages.back());
      r.pages.pop_back();
    }
  }
  std::vector<int> pend_triples;

  void admit_pending() {
    while (!pending.empty() && static_cast<int>(live.size()) < cfg.max_batch && !free_slots.empty()) {
      const int64_t id = pending.front();
      pending.pop_front();
      Req& r = reqs.at(id);
      r.slot = free_slots.back();
      free_slots.pop_back();
      live.push_back(id);
    }
  }

  // ---------------------------------------------------------------- step
  template <class T>
  T* carve(size_t& off, size_t n) {
    off = (off + 15) & ~size_t(15);
    T* p = reinterpret_cast<T*>(h_blob + off);
    off += sizeof(T) * n;
    if (off > blob_cap) throw LFail{FASER_ECAPACITY, "step blob overflow"};
    return p;
  }
  template <class T>
  T* dev_of(const T* host) const {
    return reinterpret_cast<T*>(d_blob + (reinterpret_cast<const char*>(host) - h_blob));
  }

  // PipelineTimeline of the last overlapped step (overlap.cpp:44-91 semantics, measured): event
  // times relative to the lanes' fork; a chunk with no request left on its frontier has no
  // VerifyChunk, its (not cancelled) draft counts as waste; Reset where the frontier shrank.
  void build_timeline() {
    const int nch = tl_nch;
    const int32_t* rec = h_lane;
    const int32_t* dec = h_lane + kLaneRec;
    const int32_t* res = dec + kLaneDec;
    auto at = [&](cudaEvent_t e) {
      float ms = 0.f;
      LCK(cudaEventElapsedTime(&ms, ev_fork, e));
      return static_cast<double>(ms);
    };
    faser_timeline_info& I = tl_info;
    I = faser_timeline_info{};
    tl_events.clear();
    I.n_chunks = nch;
    I.draft_sms = tl_lp.draft_sms;
    I.verify_sms = tl_lp.verify_sms;
    I.green = tl_lp.green ? 1 : 0;
    I.lane_mode = tl_lane_mode;
    for (int t = 0; t < kLaneDec; ++t) I.cancelled_draft_steps += dec[t] == 2;
    for (int qq = 0; qq < nch && qq <= FASER_MAX_SPEC; ++qq) {
      I.chunk_alive[qq] = rec[2 * qq];
      I.chunk_rows[qq] = rec[2 * qq + 1];
      I.chunk_resets[qq] = res[qq];
    }
    I.survivors = rec[2 * nch];
    for (int qq = 0; qq < nch; ++qq) {
      const double d0 = at(ev_d0[qq]), d1 = at(ev_d1[qq]);
      const double v0 = at(ev_v0[qq]), v1 = at(ev_v1[qq]);
      const int alive = rec[2 * qq];
      if (d1 - d0 > 1e-3) {  // a chunk whose steps were all cancelled ran no kernels worth timing
        tl_events.push_back({FASER_EV_DRAFT_CHUNK, qq, d0, d1});
        I.draft_busy_ms += d1 - d0;
        if (alive == 0) I.wasted_draft_ms += d1 - d0;
      }
      if (alive > 0) {
        tl_events.push_back({FASER_EV_VERIFY_CHUNK, qq, v0, v1});
        I.verify_busy_ms += v1 - v0;
        if (res[qq] > 0) tl_events.push_back({FASER_EV_RESET, qq, v1, v1});
      }
    }
    const double end = at(ev[2]);
    tl_events.push_back({FASER_EV_COMMIT, nch - 1, end, end});
    for (const auto& e : tl_events) I.makespan_ms = std::max(I.makespan_ms, e.end_ms);
    I.n_events = static_cast<int32_t>(tl_events.size());
  }

  double h_step_ms = 0.0, h_pfenq_ms = 0.0, h_sync_ms = 0.0, h_main_ms = 0.0;
  void step(const faser_step_plan* plan, faser_round_result* out, int cap, int* n_out) {
    Nvtx nv_step("faser.step");
    const auto hs0 = std::chrono::steady_clock::now();
    struct HAcc {
      double& acc;
      std::chrono::steady_clock::time_point t0;
      ~HAcc() { acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
    } hacc{h_step_ms, hs0};
    LCK(cudaSetDevice(cfg.device));
    admit_pending();
    // prefill-lane step: the requests whose prefill completed run; the new ones are admitted and
    // prefilled on pstream; those still prefilling sit the step out. With nothing able to run,
    // the oldest prefill is waited for; with nothing running or prefilling, the new requests are
    // prefilled and stepped serially (the plain path).
    bool lane_pf = false;
    pf_defer = false;
    if (pstream) {  // the lane exists (cfg.prefill_lane); pf_lane: currently used
      auto retire = [&](bool wait) {
        while (!pf_q.empty()) {
          const cudaEvent_t e = ev_pf_done[pf_q.front().blob];
          if (wait) {
            const auto w0 = std::chrono::steady_clock::now();
            LCK(cudaEventSynchronize(e));
            pf_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
            ++pf_waits;
            wait = false;
          } else {
            const cudaError_t q = cudaEventQuery(e);
            if (q == cudaErrorNotReady) break;
            LCK(q);
          }
          for (int64_t id : pf_q.front().ids) {
            auto it = reqs.find(id);
            if (it != reqs.end()) it->second.prefilling = false;
          }
          pf_q.pop_front();
        }
      };
      retire(false);
      while (!pf_lane && !pf_q.empty()) retire(true);  // lane switched off: drain it
      bool any_ready = false, any_fresh = false;
      for (int64_t id : live) {
        const Req& r = reqs.at(id);
        if (!r.admitted) any_fresh = true;
        else if (!r.prefilling) any_ready = true;
      }
      if (!any_ready && !pf_q.empty()) {  // nothing can run before the oldest prefill ends
        retire(true);
        retire(false);
        any_ready = true;
      }
      lane_pf = pf_lane && any_fresh && any_ready && cfg.debug_capture == 0 &&
                !(cfg.mode == FASER_MODE_FULL && plan && plan->overlap.enabled);
      // at most kPfInFlight prefill batches queued on the lane: more would fill the device's
      // launch queue and block the host's enqueue of the running batch; the new requests wait
      // (unadmitted, out of the step) until the lane drains
      pf_defer = lane_pf && static_cast<int>(pf_q.size()) >= pf_in_flight_cap;
      // this step's blob must not be read by an in-flight prefill
      blob_i = (blob_i + 1) % kBlobs;
      for (bool busy = true; busy;) {
        busy = false;
        for (const PfBatch& b : pf_q) busy |= b.blob == blob_i;
        if (busy) retire(true);
      }
      h_blob = h_blobs[blob_i];
      d_blob = d_blobs[blob_i].as<char>();
    }
    run.clear();
    for (int64_t id : live) {
      const Req& r = reqs.at(id);
      if (r.prefilling) continue;
      if (!lane_pf || r.admitted) run.push_back(id);
    }
    if (pf_defer) lane_pf = false;  // ready requests run; the new ones sit this step out
    const int n = static_cast<int>(run.size());
    *n_out = n;
    if (n == 0) return;
    if (cap < n) throw LFail{FASER_ECAPACITY, "result capacity smaller than live batch"};
    const int L = tsh.layers;
    stages.clear();
    pend_triples.clear();

    // ---- admissions (prompt -> slot row) + prefill rows
    struct Pre {
      int req_idx;  // index into live
      int rows;
    };
    std::vector<LmAdmit> admits;
    std::vector<int64_t> newly;
    if (!pf_defer)
      for (int64_t id : live)
        if (!reqs.at(id).admitted) newly.push_back(id);
    // ---- per request k' and ordering
    struct Ent {
      int live_idx, k;
    };
    std::vector<Ent> ents(n);
    int kmax = 0, total = 0, maxctx = 0;
    int64_t ctx_sum = 0;
    for (int i = 0; i < n; ++i) {
      Req& r = reqs.at(run[i]);
      const int remaining = r.max_out - static_cast<int>(r.committed.size());
      int k = std::min(r.spec, remaining);
      k = std::min(k, max_spec);
      if (k < 1) throw LFail{FASER_EILLEGAL_STATE, "draft on a finished request"};
      ents[i] = {i, k};
    }
    std::stable_sort(ents.begin(), ents.end(), [](const Ent& a, const Ent& b) { return a.k > b.k; });
    for (int i = 0; i < n; ++i) {
      Req& r = reqs.at(run[ents[i].live_idx]);
      kmax = std::max(kmax, ents[i].k);
      total += ents[i].k;
      // draft & verify write positions len-1 .. len+k-2
      ensure_pages(r, r.len + ents[i].k - 2);
      maxctx = std::max(maxctx, r.len - 1 + ents[i].k);
      ctx_sum += r.len - 1;
    }
    if (total > wt.rows_cap) throw LFail{FASER_ECAPACITY, "verify rows exceed capacity"};

    // ---- lay out the blob
    size_t off = 0;
    int32_t* b_slot = carve<int32_t>(off, n);
    int32_t* b_k = carve<int32_t>(off, n);
    int32_t* b_spec = carve<int32_t>(off, n);
    int32_t* b_live = carve<int32_t>(off, n);
    int64_t* b_id = carve<int64_t>(off, n);
    int32_t* v_nrows = carve<int32_t>(off, 4);
    int32_t* v_row_req = carve<int32_t>(off, total);
    int32_t* v_row_pos = carve<int32_t>(off, total);
    int32_t* v_row_tok = carve<int32_t>(off, total);
    int32_t* v_row_j = carve<int32_t>(off, total);
    int32_t* v_first = carve<int32_t>(off, n);
    int32_t* v_n = carve<int32_t>(off, n);
    int32_t* v_rslot = carve<int32_t>(off, n);
    int32_t* v_pos0 = carve<int32_t>(off, n);
    step_sorted_ids.resize(n);
    {
      int row = 0;
      for (int i = 0; i < n; ++i) {
        Req& r = reqs.at(run[ents[i].live_idx]);
        b_slot[i] = r.slot;
        b_k[i] = ents[i].k;
        b_spec[i] = r.spec;
        b_live[i] = ents[i].live_idx;
        b_id[i] = r.id;
        step_sorted_ids[i] = r.id;
        v_first[i] = row;
        v_n[i] = ents[i].k;
        v_rslot[i] = r.slot;
        v_pos0[i] = r.len - 1;
        for (int j = 0; j < ents[i].k; ++j, ++row) {
          v_row_req[row] = i;
          v_row_pos[row] = r.len - 1 + j;
          v_row_tok[row] = 0;
          v_row_j[row] = j;
        }
      }
      v_nrows[0] = total;
    }
    // overlapped mode: verify row sets per frontier chunk [q*c, (q+1)*c) of drafted positions
    struct VChunkH {
      int32_t *nrows, *row_req, *row_pos, *row_tok, *row_j, *first, *nn, *rslot, *pos0;
      int T, max_rows;
    };
    std::vector<VChunkH> chunks_h;
    // chunk < k: frontier-chunked overlap; chunk >= k with a share r in (0,1): one chunk, the two
    // stages back to back on their partitions (per-share stage profiling)
    const bool part_r = plan && plan->overlap.r > 0.0 && plan->overlap.r < 1.0;
    const bool overlap = cfg.mode == FASER_MODE_FULL && plan && plan->overlap.enabled &&
                         plan->overlap.chunk >= 1 && (plan->overlap.chunk < kmax || part_r) && !use_graph_mode();
    if (overlap) {
      const int c = std::min(plan->overlap.chunk, kmax);
      for (int q0 = 0; q0 < kmax; q0 += c) {
        int T = 0;
        for (int i = 0; i < n; ++i) T += std::max(0, std::min(ents[i].k, q0 + c) - q0);
        VChunkH h;
        h.T = T;
        h.max_rows = std::min(c, kmax - q0);
        h.nrows = carve<int32_t>(off, 4);
        h.row_req = carve<int32_t>(off, T);
        h.row_pos = carve<int32_t>(off, T);
        h.row_tok = carve<int32_t>(off, T);
        h.row_j = carve<int32_t>(off, T);
        h.first = carve<int32_t>(off, n);
        h.nn = carve<int32_t>(off, n);
        h.rslot = carve<int32_t>(off, n);
        h.pos0 = carve<int32_t>(off, n);
        int row = 0;
        for (int i = 0; i < n; ++i) {
          Req& r = reqs.at(run[ents[i].live_idx]);
          const int j1 = std::min(ents[i].k, q0 + c);
          h.first[i] = row;
          h.nn[i] = std::max(0, j1 - q0);
          h.rslot[i] = r.slot;
          h.pos0[i] = r.len - 1 + q0;
          for (int j = q0; j < j1; ++j, ++row) {
            h.row_req[row] = i;
            h.row_pos[row] = r.len - 1 + j;
            h.row_tok[row] = 0;
            h.row_j[row] = j;
          }
        }
        h.nrows[0] = T;
        chunks_h.push_back(h);
      }
    }
    // lane state of the overlapped mode (LaneState): rec | step_dec | alive, zero except alive = n
    int32_t* b_rec = carve<int32_t>(off, kLaneInts);
    std::memset(b_rec, 0, sizeof(int32_t) * kLaneInts);
    int32_t* b_dec = b_rec + kLaneRec;
    int32_t* b_res = b_dec + kLaneDec;
    int32_t* b_alive = b_res + kLaneRes;
    *b_alive = n;
    // admissions: slot row copy + page reservation for the prompt prefix
    for (int64_t id : newly) {
      Req& r = reqs.at(id);
      if (r.len >= 2) ensure_pages(r, r.len - 2);
    }
    int32_t* b_tr = carve<int32_t>(off, pend_triples.size());
    std::memcpy(b_tr, pend_triples.data(), pend_triples.size() * 4);
    const int n_tr = static_cast<int>(pend_triples.size() / 3);
    // prompts: staged in the blob itself
    std::vector<std::pair<int32_t*, int64_t>> prompt_at;
    for (int64_t id : newly) {
      Req& r = reqs.at(id);
      int32_t* pr = carve<int32_t>(off, r.prompt.size());
      std::memcpy(pr, r.prompt.data(), r.prompt.size() * 4);
      prompt_at.push_back({pr, id});
    }
    LmAdmit* b_adm = carve<LmAdmit>(off, newly.size());
    for (size_t i = 0; i < newly.size(); ++i) {
      Req& r = reqs.at(newly[i]);
      b_adm[i].src = dev_of(prompt_at[i].first);
      b_adm[i].slot = r.slot;
      b_adm[i].len = static_cast<int>(r.prompt.size());
      b_adm[i].max_out = r.max_out;
      b_adm[i].reserved = 0;
    }
    // prefill chunks (rows = prompt positions 0..len-2 of newly admitted requests)
    struct Chunk {
      int32_t *nrows, *row_req, *row_pos, *row_tok, *row_j, *first, *nn, *rslot, *pos0;
      int T, nreq, maxrows, maxctx;
    };
    std::vector<Chunk> chunks;
    {
      const int cap_rows = std::min(wt.rows_cap, wd.rows_cap);
      size_t i = 0;
      while (i < newly.size()) {
        std::vector<int64_t> grp;
        int rows = 0;
        while (i < newly.size()) {
          const int rr = reqs.at(newly[i]).len - 1;
          if (rr <= 0) {
            ++i;
            continue;
          }
          if (rows + rr > cap_rows && !grp.empty()) break;
          grp.push_back(newly[i]);
          rows += rr;
          ++i;
        }
        if (grp.empty()) continue;
        Chunk c;
        c.T = rows;
        c.nreq = static_cast<int>(grp.size());
        c.nrows = carve<int32_t>(off, 4);
        c.row_req = carve<int32_t>(off, rows);
        c.row_pos = carve<int32_t>(off, rows);
        c.row_tok = carve<int32_t>(off, rows);
        c.row_j = carve<int32_t>(off, rows);
        c.first = carve<int32_t>(off, grp.size());
        c.nn = carve<int32_t>(off, grp.size());
        c.rslot = carve<int32_t>(off, grp.size());
        c.pos0 = carve<int32_t>(off, grp.size());
        c.maxrows = 0;
        c.maxctx = 0;
        int row = 0;
        for (size_t g = 0; g < grp.size(); ++g) {
          Req& r = reqs.at(grp[g]);
          const int rr = r.len - 1;
          c.first[g] = row;
          c.nn[g] = rr;
          c.rslot[g] = r.slot;
          c.pos0[g] = 0;
          c.maxrows = std::max(c.maxrows, rr);
          c.maxctx = std::max(c.maxctx, rr);
          for (int j = 0; j < rr; ++j, ++row) {
            c.row_req[row] = static_cast<int>(g);
            c.row_pos[row] = j;
            c.row_tok[row] = 0;
            c.row_j[row] = j;
          }
        }
        c.nrows[0] = rows;
        chunks.push_back(c);
      }
    }
    const size_t blob_bytes = off;
    LCK(cudaMemcpyAsync(d_blob, h_blob, blob_bytes, cudaMemcpyHostToDevice, stream));
    h2d = static_cast<int64_t>(blob_bytes);
    d2h = static_cast<int64_t>(sizeof(faser_round_result)) * n;

    std::vector<VChunk> chunks_v;
    for (const VChunkH& h : chunks_h) {
      VChunk v;
      v.T = h.T;
      v.max_rows = h.max_rows;
      v.rows.n_rows = dev_of(h.nrows);
      v.rows.row_req = dev_of(h.row_req);
      v.rows.row_pos = dev_of(h.row_pos);
      v.rows.row_tok = dev_of(h.row_tok);
      v.rows.row_j = dev_of(h.row_j);
      v.rows.req_first = dev_of(h.first);
      v.rows.req_n = dev_of(h.nn);
      v.rows.req_slot = dev_of(h.rslot);
      v.rows.req_pos0 = dev_of(h.pos0);
      chunks_v.push_back(v);
    }
    LmReqState q = rq;
    q.slot = dev_of(b_slot);
    q.k = dev_of(b_k);
    q.spec = dev_of(b_spec);
    q.live_idx = dev_of(b_live);
    q.req_id = dev_of(b_id);
    cur_q = q;
    RowsDev vrows;
    vrows.n_rows = dev_of(v_nrows);
    vrows.row_req = dev_of(v_row_req);
    vrows.row_pos = dev_of(v_row_pos);
    vrows.row_tok = dev_of(v_row_tok);
    vrows.row_j = dev_of(v_row_j);
    vrows.req_first = dev_of(v_first);
    vrows.req_n = dev_of(v_n);
    vrows.req_slot = dev_of(v_rslot);
    vrows.req_pos0 = dev_of(v_pos0);

    const bool use_graph = graph_mode && cfg.debug_capture == 0;
    if (use_graph) {
      LCK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      capturing = true;
    }
    LCK(record_event(ev[0]));
    nvtxRangePushA("faser.admit_prefill");
    LCK(lm_ptab_scatter(ptab.as<int>(), max_pages, dev_of(b_tr), n_tr, stream));
    LCK(lm_admit(sl, dev_of(b_adm), static_cast<int>(newly.size()), stream));
    launches += (n_tr > 0) + (!newly.empty());
    // admission prefill forwards on stream `ps`: in the step (serial) or on the prefill lane,
    // where they are enqueued after the running batch's work so the host's launch time for
    // them never delays the batch
    auto enqueue_prefill = [&](cudaStream_t ps) {
    for (const Chunk& c : chunks) {
      RowsDev pr;
      pr.n_rows = dev_of(c.nrows);
      pr.row_req = dev_of(c.row_req);
      pr.row_pos = dev_of(c.row_pos);
      pr.row_tok = dev_of(c.row_tok);
      pr.row_j = dev_of(c.row_j);
      pr.req_first = dev_of(c.first);
      pr.req_n = dev_of(c.nn);
      pr.req_slot = dev_of(c.rslot);
      pr.req_pos0 = dev_of(c.pos0);
      LCK(lm_prefill_tokens(sl, pr, c.T, ps));
      ++launches;
      Fwd f;
      f.rows = pr;
      f.T = c.T;
      f.n_req = c.nreq;
      f.max_rows = c.maxrows;
      f.max_ctx = c.maxctx;
      fs = ps;  // (fs may still name the verify lane of the previous overlapped step)
      forward(draft, ps == stream ? wd : wd_pf, f);
      forward(target, ps == stream ? wt : wt_pf, f);
    }
    fs = stream;
    };
    const bool pf_on_lane = lane_pf && !chunks.empty();
    if (pf_on_lane) {
      LCK(cudaEventRecord(ev_pf_go, stream));  // slot rows + page table written
      LCK(cudaStreamWaitEvent(pstream, ev_pf_go, 0));
    } else {
      enqueue_prefill(stream);
    }
    LCK(record_event(ev[3]));  // end of admission + prefill
    nvtxRangePop();  // faser.admit_prefill
    // ---- early-exit configuration
    const bool capture = cfg.debug_capture != 0;
    const bool ee = cfg.mode >= FASER_MODE_VSD_AD_EE;
    int k_table[FASER_MAX_LAYERS + 1];
    int glo = 0, ghi = 0;
    if (ee) {
      faser_gate_plan g{cfg.exit_policy.l_init, cfg.exit_policy.l_init, 1.0};
      if (plan) g = plan->gate;
      glo = std::max(g.first_layer, 1);
      ghi = std::min(g.stop_layer, L);
      if (!(g.first_layer < g.stop_layer)) glo = ghi = 0;
      if (plan && plan->use_k_table) {
        for (int l = 0; l <= L; ++l) {
          if (plan->k_table[l] < 1) throw LFail{FASER_EINVAL, "k must be >= 1"};
          k_table[l] = plan->k_table[l];
        }
      } else if (faser_k_table(&cfg.exit_policy, L, k_table) != FASER_OK) {
        throw LFail{FASER_EINVAL, "invalid exit policy"};
      }
    }
    // fused draft control (one launch between draft forwards)
    const bool fuse_draft = !(getenv("FASER_UNFUSED_DRAFT") && getenv("FASER_UNFUSED_DRAFT")[0] == '1');
    // verify: tokens + embedding in one launch, argmax + truth scatter in one launch (not under
    // TP, whose argmax is the all-gathered merge, nor with the persistent forward)
    const bool fuse_verify = fuse_draft && tp == 1;
    auto rows_at = [&](int t) {
      int c = 0;
      while (c < n && ents[c].k > t) ++c;
      return c;
    };
    // lanes: the draft lane drafts, the verify lane verifies; serial mode runs both on `stream`.
    // Overlapped (FULL) mode with overlap.r in (0,1) puts them on disjoint green-context SM
    // partitions (lanes.cuh) and the GEMM plans size their grids for the lane's SM count.
    LanePair lp;
    lp.draft = lp.verify = stream;
    lp.draft_sms = lp.verify_sms = nsm;
    if (overlap) {
      if (plan->overlap.r > 0.0 && plan->overlap.r < 1.0) {
        if (!lanes) lanes = std::make_unique<SmLanes>(cfg.device, nsm);
        std::string lerr;
        if (!lanes->get(plan->overlap.r, &lp, &lerr)) throw LFail{FASER_ECUDA, lerr};
      } else {
        lp.verify = vstream;
      }
    }
    const cudaStream_t ds = lp.draft;
    auto draft_step = [&](int t, const LaneState* ln) {
      const int nt = rows_at(t);
      fwd_sms = lp.draft_sms;
      if (fuse_draft) {
        if (t == 0) {
          LCK(lm_draft_begin(sl, q, wd.rows, nt, draft.emb, dsh.d, wd.x.as<float>(), wd.xb.as<__nv_bfloat16>(),
                             wd.ss.as<float>(), ds));
          ++launches;
        }
        Fwd f;
        f.rows = wd.rows;
        f.T = nt;
        f.n_req = nt;
        f.max_rows = 1;
        f.max_ctx = maxctx;
        f.logits = true;
        f.argmax_out = wd.argmax.as<int>();
        f.kv_tokens = ctx_sum + static_cast<int64_t>(nt) * (t + 1);
        f.pre_embedded = true;
        f.skip_argmax = true;
        fs = ds;
        forward(draft, wd, f);
        const int n_next = t + 1 < kmax ? rows_at(t + 1) : 0;
        LCK(lm_draft_advance(sl, q, wd.rows, wd.amax.as<float2>(), dsh.vocab / 128, nt, t, n_next, draft.emb, dsh.d,
                             wd.x.as<float>(), wd.xb.as<__nv_bfloat16>(), wd.ss.as<float>(), ds, ln));
        ++launches;
        return;
      }
      LCK(lm_draft_prep(sl, q, wd.rows, nt, t, ds));
      Fwd f;
      f.rows = wd.rows;
      f.T = nt;
      f.n_req = nt;
      f.max_rows = 1;
      f.max_ctx = maxctx;
      f.logits = true;
      f.argmax_out = wd.argmax.as<int>();
      f.kv_tokens = ctx_sum + static_cast<int64_t>(nt) * (t + 1);
      fs = ds;
      forward(draft, wd, f);
      LCK(lm_draft_post(q, wd.argmax.as<int>(), nt, t, ds));
      launches += 2;
    };
    cudaStream_t vs = stream;  // stream of the verify lane
    tl_valid = false;
    if (!chunks_v.empty()) {
      // ---- overlapped (FULL) mode: frontier chunk q is verified on the verify lane while the
      // draft lane drafts chunk q+1 (overlap.cpp:44-91 made real). Before each chunk the verify
      // lane drops the requests whose frontier was reset by an earlier chunk (rejection, prune
      // or EOS): their rows are cancelled, and once no request is left the draft lane cancels
      // the steps it has not started. Early exit runs inside every chunk (FULL = AD + EE +
      // overlap); truth is scattered per (request, position) for the accept.
      vs = lp.verify;
      const int c = std::min(plan->overlap.chunk, kmax);
      const int nch = static_cast<int>(chunks_v.size());
      const bool isolate = plan->lane_mode == 1;
      LaneState ln{dev_of(b_alive), dev_of(b_rec), dev_of(b_dec), dev_of(b_res)};
      LCK(cudaEventRecord(ev_fork, stream));
      LCK(cudaStreamWaitEvent(ds, ev_fork, 0));
      if (vs != ds) LCK(cudaStreamWaitEvent(vs, ev_fork, 0));
      for (int qi = 0; qi < nch; ++qi) {
        if (isolate && qi > 0 && vs != ds) LCK(cudaStreamWaitEvent(ds, ev_v1[qi - 1], 0));
        LCK(cudaEventRecord(ev_d0[qi], ds));
        for (int t = qi * c; t < std::min(kmax, (qi + 1) * c); ++t) draft_step(t, fuse_draft ? &ln : nullptr);
        LCK(cudaEventRecord(ev_d1[qi], ds));
        if (qi + 1 == nch) LCK(cudaEventRecord(ev[1], ds));
        LCK(cudaEventRecord(ev_chunk[qi], ds));
        LCK(cudaStreamWaitEvent(vs, ev_chunk[qi], 0));
        LCK(cudaEventRecord(ev_v0[qi], vs));
        const VChunk& vc = chunks_v[qi];
        LCK(lm_chunk_frontier(q, vc.rows, n, qi, qi * c, qi == 0 ? 1 : 0, L, eos, ln, vs));
        Fwd f;
        if (fuse_verify) {
          LCK(lm_verify_begin(sl, q, vc.rows, vc.T, target.emb, tsh.d, wt.x.as<float>(), wt.xb.as<__nv_bfloat16>(),
                              wt.ss.as<float>(), vs));
          f.pre_embedded = f.skip_argmax = true;
        } else {
          LCK(lm_verify_tokens(sl, q, vc.rows, vc.T, vs));
        }
        f.rows = vc.rows;
        f.T = vc.T;
        f.n_req = n;
        f.max_rows = vc.max_rows;
        f.max_ctx = maxctx;
        f.logits = true;
        f.argmax_out = rq.truth;
        f.kv_tokens = ctx_sum + vc.T;
        f.ee = ee;
        f.gate_lo = glo;
        f.gate_hi = ghi;
        f.k_table = k_table;
        f.q0 = qi * c;
        fs = vs;
        fwd_sms = lp.verify_sms;
        forward(target, wt, f);
        if (fuse_verify)
          LCK(lm_verify_argmax(vc.rows, target.sh.vocab / 128, vc.T, wt.amax.as<float2>(), rq.truth, rq.truth_rj, vs));
        else
          LCK(lm_truth_scatter(vc.rows, rq.truth, rq.truth_rj, vc.T, vs));
        LCK(cudaEventRecord(ev_v1[qi], vs));
        launches += 3;
      }
      LCK(lm_chunk_finalize(q, n, eos, nch, c, ln, vs));
      ++launches;
      tl_nch = nch;
      tl_lane_mode = isolate ? 1 : 0;
      tl_lp = lp;
      tl_valid = true;
    } else {
      nvtxRangePushA("faser.draft");
      for (int t = 0; t < kmax; ++t) draft_step(t, nullptr);
      nvtxRangePop();
      LCK(record_event(ev[1]));
      // ---- verify (+ early exit)
      Nvtx nv_verify("faser.verify");
      LCK(lm_verify_init(q, n, L, eos, stream));
      Fwd f;
      if (fuse_verify) {
        LCK(lm_verify_begin(sl, q, vrows, total, target.emb, tsh.d, wt.x.as<float>(), wt.xb.as<__nv_bfloat16>(),
                            wt.ss.as<float>(), stream));
        f.pre_embedded = f.skip_argmax = true;
      } else {
        LCK(lm_verify_tokens(sl, q, vrows, total, stream));
      }
      f.rows = vrows;
      f.T = total;
      f.n_req = n;
      f.max_rows = kmax;
      f.max_ctx = maxctx;
      f.logits = true;
      f.argmax_out = rq.truth;
      f.kv_tokens = ctx_sum + total;
      f.ee = ee;
      f.gate_lo = glo;
      f.gate_hi = ghi;
      f.k_table = k_table;
      f.capture = capture;
      fs = stream;
      forward(target, wt, f);
      if (fuse_verify)
        LCK(lm_verify_argmax(vrows, target.sh.vocab / 128, total, wt.amax.as<float2>(), rq.truth, rq.truth_rj, stream));
      else
        LCK(lm_truth_scatter(vrows, rq.truth, rq.truth_rj, total, stream));
      launches += 3;
    }
    fwd_sms = nsm;
    StepCtl ctl{n, L, eos, ee ? 1 : 0, cfg.exempt_rule};
    LCK(lm_accept_commit(sl, q, vrows, ctl, d_res.as<faser_round_result>(), vs));
    ++launches;
    if (vs == stream)
      LCK(record_event(ev[2]));
    else
      LCK(cudaEventRecord(ev[2], vs));
    if (vs != stream) LCK(cudaStreamWaitEvent(stream, ev[2], 0));
    if (ds != stream) {  // join the draft lane too: the next step's blob upload must not race it
      LCK(cudaEventRecord(ev_dend, ds));
      LCK(cudaStreamWaitEvent(stream, ev_dend, 0));
    }
    h_main_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hs0).count();
    if (pf_on_lane) {  // the admissions' prefill, behind the batch's work in host order
      const auto e0 = std::chrono::steady_clock::now();
      enqueue_prefill(pstream);
      h_pfenq_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - e0).count();
      LCK(cudaEventRecord(ev_pf_done[blob_i], pstream));
      pf_q.push_back({blob_i, newly});
      for (int64_t id : newly) reqs.at(id).prefilling = true;
    }
    if (use_graph) {
      capturing = false;
      cudaGraph_t g = nullptr;
      LCK(cudaStreamEndCapture(stream, &g));
      cudaGraphExec_t ge = nullptr;
      LCK(cudaGraphInstantiate(&ge, g, 0));
      LCK(cudaGraphLaunch(ge, stream));
      LCK(cudaStreamSynchronize(stream));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
    LCK(cudaMemcpyAsync(h_res, d_res.p, sizeof(faser_round_result) * n, cudaMemcpyDeviceToHost, stream));
    if (tl_valid)
      LCK(cudaMemcpyAsync(h_lane, dev_of(b_rec), sizeof(int32_t) * kLaneInts, cudaMemcpyDeviceToHost, stream));
    if (capture) {
      std::vector<int32_t> dr(static_cast<size_t>(n) * FASER_MAX_SPEC);
      LCK(cudaMemcpyAsync(dr.data(), rq.drafted, dr.size() * 4, cudaMemcpyDeviceToHost, stream));
      LCK(cudaStreamSynchronize(stream));
      dbg_drafted.assign(dr.size(), 0);
      for (int i = 0; i < n; ++i)
        std::memcpy(&dbg_drafted[static_cast<size_t>(ents[i].live_idx) * FASER_MAX_SPEC],
                    &dr[static_cast<size_t>(i) * FASER_MAX_SPEC], FASER_MAX_SPEC * 4);
    }
    {
      const auto s0 = std::chrono::steady_clock::now();
      LCK(cudaStreamSynchronize(stream));
      h_sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s0).count();
    }
    if (ktiming) resolve_kernel_timing();
    cudaEventElapsedTime(&t_draft, ev[0], ev[1]);
    cudaEventElapsedTime(&t_prefill, ev[0], ev[3]);
    cudaEventElapsedTime(&t_verify, ev[1], ev[2]);
    cudaEventElapsedTime(&t_step, ev[0], ev[2]);
    if (tl_valid) build_timeline();

    // ---- host bookkeeping: commit mirror, page rollback, retire finished requests
    for (int64_t id : newly) reqs.at(id).admitted = true;
    std::vector<int64_t> keep;
    keep.reserve(live.size());
    if (pf_lane)  // prefilling on the lane or deferred: drafted from a later step
      for (int64_t id : live)
        if (reqs.at(id).prefilling || (pf_defer && !reqs.at(id).admitted)) keep.push_back(id);
    for (int p = 0; p < n; ++p) {
      const faser_round_result& rr = h_res[p];
      Req& r = reqs.at(run[p]);
      r.committed.insert(r.committed.end(), rr.tokens, rr.tokens + rr.committed);
      r.len += rr.committed;
      r.done = rr.done != 0;
      if (r.done) {
        release_pages_beyond(r, 0);
        free_slots.push_back(r.slot);
        r.slot = -1;
      } else {
        // the cache must hold positions [0, len-1): pages 0 .. (len-2)/64
        release_pages_beyond(r, r.len >= 2 ? (r.len - 2) / kPage + 1 : 0);
        keep.push_back(r.id);
      }
    }
    std::memcpy(out, h_res, sizeof(faser_round_result) * n);
    live.swap(keep);
  }
};

// ------------------------------------------------------------------ C-side wrappers
namespace {
template <class F>
faser_status lguard(LlamaEngine* e, F&& f) {
  try {
    f();
    return FASER_OK;
  } catch (const LFail& x) {
    if (e) e->err = x.msg;
    return x.st;
  } catch (const std::bad_alloc&) {
    if (e) e->err = "host allocation failed";
    return FASER_ENOMEM;
  }
}
thread_local std::string g_create_err;
}  // namespace

LlamaEngine* llama_engine_create(const faser_model_desc* model, const faser_engine_cfg* cfg,
                                 faser_status* st, const char** msg) {
  LlamaEngine* e = new LlamaEngine();
  try {
    e->create(model, cfg);
    *st = FASER_OK;
    return e;
  } catch (const LFail& x) {
    g_create_err = x.msg;
    *st = x.st;
  } catch (const std::bad_alloc&) {
    g_create_err = "host allocation failed";
    *st = FASER_ENOMEM;
  }
  *msg = g_create_err.c_str();
  delete e;
  return nullptr;
}

void llama_engine_destroy(LlamaEngine* e) { delete e; }
const char* llama_last_error(const LlamaEngine* e) { return e->err.c_str(); }

faser_status llama_submit(LlamaEngine* e, int64_t req_id, const int32_t* prompt, int32_t len, int32_t max_out) {
  return lguard(e, [&] {
    if (!prompt || len < 1) throw LFail{FASER_EINVAL, "prompt must be non-empty"};
    if (max_out < 0) throw LFail{FASER_EINVAL, "max_out must be >= 0"};
    if (e->reqs.count(req_id)) throw LFail{FASER_EINVAL, "duplicate request id"};
    if (static_cast<int64_t>(len) + max_out > e->cfg.max_seq_len)
      throw LFail{FASER_ECAPACITY, "prompt + max_out exceeds max_seq_len"};
    for (int i = 0; i < len; ++i)
      if (prompt[i] < 0 || prompt[i] >= e->tsh.vocab) throw LFail{FASER_EINVAL, "token outside vocabulary"};
    LlamaEngine::Req r;
    r.id = req_id;
    r.prompt.assign(prompt, prompt + len);
    r.max_out = max_out;
    r.spec = e->cfg.default_spec_length;
    r.len = len;
    r.done = max_out == 0;
    e->reqs.emplace(req_id, std::move(r));
    if (max_out > 0) e->pending.push_back(req_id);
  });
}

faser_status llama_set_spec_lengths(LlamaEngine* e, const int64_t* ids, const int32_t* k, int32_t n) {
  return lguard(e, [&] {
    for (int i = 0; i < n; ++i) {
      if (k[i] < 1 || k[i] > e->max_spec) throw LFail{FASER_EINVAL, "speculative length must be in [1, max_spec_length]"};
      auto it = e->reqs.find(ids[i]);
      if (it == e->reqs.end()) throw LFail{FASER_EINVAL, "unknown request id"};
      it->second.spec = k[i];
    }
  });
}

faser_status llama_live_requests(LlamaEngine* e, int64_t* ids, int32_t cap, int32_t* n) {
  return lguard(e, [&] {
    e->admit_pending();
    *n = static_cast<int32_t>(e->live.size());
    for (int i = 0; i < *n && i < cap; ++i) ids[i] = e->live[i];
  });
}

faser_status llama_step(LlamaEngine* e, const faser_step_plan* plan, faser_round_result* out, int32_t cap,
                        int32_t* n_out) {
  return lguard(e, [&] { e->step(plan, out, cap, n_out); });
}

faser_status llama_get_committed(LlamaEngine* e, int64_t req_id, int32_t* buf, int32_t cap, int32_t* n) {
  return lguard(e, [&] {
    auto it = e->reqs.find(req_id);
    if (it == e->reqs.end()) throw LFail{FASER_EINVAL, "unknown request id"};
    const auto& c = it->second.committed;
    *n = static_cast<int32_t>(c.size());
    if (buf) std::memcpy(buf, c.data(), sizeof(int32_t) * std::min<size_t>(c.size(), std::max(cap, 0)));
  });
}

faser_status llama_release(LlamaEngine* e, int64_t req_id) {
  return lguard(e, [&] {
    auto it = e->reqs.find(req_id);
    if (it == e->reqs.end()) throw LFail{FASER_EINVAL, "unknown request id"};
    if (!it->second.done) throw LFail{FASER_EILLEGAL_STATE, "release of a live request"};
    e->reqs.erase(it);
  });
}

int32_t llama_pending_work(const LlamaEngine* e) { return static_cast<int32_t>(e->live.size() + e->pending.size()); }
faser_status llama_last_timeline(const LlamaEngine* e, faser_timeline_event* ev, int32_t cap, faser_timeline_info* info) {
  if (!e->tl_valid) return FASER_EINVAL;
  *info = e->tl_info;
  const int n = std::min<int>(cap, static_cast<int>(e->tl_events.size()));
  for (int i = 0; i < n; ++i) ev[i] = e->tl_events[i];
  return FASER_OK;
}

float llama_last_step_prefill(const LlamaEngine* e) { return e->t_prefill; }
faser_status llama_set_skip_mask(LlamaEngine* e, int mask) {
  return lguard(e, [&] { e->skip_mask = mask; });
}
faser_status llama_set_sampling(LlamaEngine* e, double temperature, uint64_t seed) {
  return lguard(e, [&] {
    if (!(temperature >= 0.0) || !std::isfinite(temperature)) throw LFail{FASER_EINVAL, "temperature must be >= 0"};
    if (temperature > 0.0 && e->cfg.mode == FASER_MODE_FULL)
      throw LFail{FASER_EINVAL, "sampling is not wired into the chunked (FULL) verify lanes"};
    e->samp_inv_tau = temperature > 0.0 ? static_cast<float>(1.0 / temperature) : 0.f;
    e->samp_seed = seed;
  });
}
faser_status llama_set_prefill_lane(LlamaEngine* e, int on) {
  return lguard(e, [&] {
    if (on && !e->pstream) throw LFail{FASER_EINVAL, "the engine was created without prefill_lane"};
    e->pf_lane = on != 0;
  });
}
faser_status llama_join_lanes(LlamaEngine* e) {
  return lguard(e, [&] {
    if (!e->pf_q.empty()) LCK(cudaStreamWaitEvent(e->stream, e->ev_pf_done[e->pf_q.back().blob], 0));
  });
}
void llama_last_step_timing(const LlamaEngine* e, float* d, float* v, float* s) {
  if (d) *d = e->t_draft;
  if (v) *v = e->t_verify;
  if (s) *s = e->t_step;
}
void llama_last_step_bytes(const LlamaEngine* e, int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = e->h2d;
  if (d2h) *d2h = e->d2h;
}
void* llama_stream(const LlamaEngine* e) { return e->stream; }
int64_t llama_launches(const LlamaEngine* e) { return e->launches; }

faser_status llama_debug_verify_logits(LlamaEngine* e, int32_t stage, float* logits, int64_t* row_ids,
                                       int32_t cap_rows, int32_t* rows) {
  return lguard(e, [&] {
    auto it = e->stages.find(stage);
    if (it == e->stages.end()) throw LFail{FASER_EINVAL, "stage not captured in the last step"};
    const auto& st = it->second;
    *rows = st.rows;
    const int n = std::min(st.rows, cap_rows);
    const size_t V = static_cast<size_t>(e->tsh.vocab);
    if (logits) std::memcpy(logits, st.logits.data(), n * V * 4);
    if (row_ids) std::memcpy(row_ids, st.ids.data(), static_cast<size_t>(n) * 2 * 8);
  });
}

faser_status llama_debug_drafted(LlamaEngine* e, int32_t* drafted, int32_t cap, int32_t* n) {
  return lguard(e, [&] {
    const int m = static_cast<int>(e->dbg_drafted.size() / FASER_MAX_SPEC);
    *n = m;
    if (drafted) std::memcpy(drafted, e->dbg_drafted.data(), static_cast<size_t>(std::min(m, cap)) * FASER_MAX_SPEC * 4);
  });
}

faser_status llama_debug_kv_pages(LlamaEngine* e, int64_t req_id, int32_t* pages, int32_t cap, int32_t* n) {
  return lguard(e, [&] {
    auto it = e->reqs.find(req_id);
    if (it == e->reqs.end()) throw LFail{FASER_EINVAL, "unknown request id"};
    const auto& p = it->second.pages;
    *n = static_cast<int32_t>(p.size());
    if (pages) std::memcpy(pages, p.data(), sizeof(int32_t) * std::min<size_t>(p.size(), std::max(cap, 0)));
  });
}

}  // namespace faser

namespace faser {
faser_status llama_debug_weights(LlamaEngine* e, int32_t model, int32_t which, int32_t layer, int64_t offset,
                                 int32_t n, uint16_t* out) {
  return lguard(e, [&] {
    if (model < 0 || model > 1 || which < 0 || which > 5 || n < 0 || !out) throw LFail{FASER_EINVAL, "bad tensor"};
    const LmModel& m = model == 0 ? e->draft : e->target;
    const LlamaShape& s = m.sh;
    if (which >= 2 && (layer < 0 || layer >= s.layers)) throw LFail{FASER_EINVAL, "layer out of range"};
    const int64_t d = s.d, qd = static_cast<int64_t>(s.n_q) * s.hd;
    const void* base = nullptr;
    int64_t size = 0;
    switch (which) {
      case 0: base = m.lm; size = static_cast<int64_t>(s.vocab) * d; break;
      case 1: base = m.emb; size = static_cast<int64_t>(s.vocab) * d; break;
      case 2: base = m.lw[layer].wqkv; size = static_cast<int64_t>(s.qkv_out()) * d; break;
      case 3: base = m.lw[layer].wo; size = d * qd; break;
      case 4: base = m.lw[layer].wgu; size = 2ll * s.ffn * d; break;
      default: base = m.lw[layer].wd; size = d * s.ffn; break;
    }
    if (offset < 0 || offset + n > size) throw LFail{FASER_EINVAL, "range outside tensor"};
    LCK(cudaMemcpy(out, static_cast<const uint16_t*>(base) + offset, static_cast<size_t>(n) * 2, cudaMemcpyDeviceToHost));
  });
}
}  // namespace faser

namespace faser {
faser_status llama_set_kernel_timing(LlamaEngine* e, int32_t on) {
  return lguard(e, [&] {
    e->ktiming = on != 0;
    for (int c = 0; c < LlamaEngine::kClasses; ++c) {
      e->k_ms[c] = e->k_bytes[c] = e->k_flops[c] = 0.0;
      e->k_n[c] = 0;
    }
  });
}
faser_status llama_kernel_stats(LlamaEngine* e, int32_t cls, double* ms, int64_t* launches, double* bytes) {
  return lguard(e, [&] {
    if (cls < 0 || cls >= LlamaEngine::kClasses) throw LFail{FASER_EINVAL, "unknown kernel class"};
    if (ms) *ms = e->k_ms[cls];
    if (launches) *launches = e->k_n[cls];
    if (bytes) *bytes = e->k_bytes[cls];
  });
}
faser_status llama_kernel_flops(LlamaEngine* e, int32_t cls, double* flops) {
  return lguard(e, [&] {
    if (cls < 0 || cls >= LlamaEngine::kClasses) throw LFail{FASER_EINVAL, "unknown kernel class"};
    if (flops) *flops = e->k_flops[cls];
  });
}
}  // namespace faser

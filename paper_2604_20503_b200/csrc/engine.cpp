// engine.cpp — C++ host engine behind include/faser/engine.h.
//
// Replaces the reference's in-process C++ path (SpeculativeEngine + Request, sdcore.hpp:39-116,
// driven by the missing serving loop) with a GPU-resident one:
//   * request table + iteration-boundary admission (B_max slots, FIFO),
//   * per-step ragged batch {slot, k_i} uploaded in ONE pinned H2D copy,
//   * draft kernel -> fused verify/accept/commit kernel on the engine stream,
//   * ONE D2H copy of the per-request round results, host mirror of committed tokens.
// Device memory (slot rows, hash states, draft scratch) is owned by the engine. There is no
// CPU compute fallback: every failing CUDA call surfaces as FASER_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "faser/engine.h"
#include "llama_engine.cuh"
#include "toy_kernels.cuh"

namespace faser {
namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;
uint64_t mix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t substream(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }

thread_local std::string g_last_error;

struct Fail {
  faser_status st;
  std::string msg;
};

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw Fail{FASER_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};       \
  } while (0)

bool valid_toy(const faser_toy_params* p, std::string* why) {
  if (!p) return *why = "null model params", false;
  if (p->vocab < 2) return *why = "vocab must be >= 2", false;
  if (p->layers < 1 || p->layers > FASER_MAX_LAYERS) return *why = "layers out of range", false;
  if (p->order < 1) return *why = "order must be >= 1", false;
  if (p->divergence < 0.0 || p->divergence > 1.0) return *why = "divergence must lie in [0,1]", false;
  if (!toy_vocab_supported(p->vocab)) return *why = "toy vocab > 256 not supported on device", false;
  return true;
}

ToyDev make_toy(const faser_toy_params& p) {
  ToyDev m{};
  m.table_seed = substream(p.seed, 0x7461626cull);  // "tabl" (toylm.cpp:23)
  m.noise_seed = substream(p.noise_seed, 0x6e6f6973ull);
  m.mix_seed = substream(p.seed, 0x6d697875ull);
  m.divergence = p.divergence;
  m.logit_scale = p.logit_scale;
  m.noise_scale = p.noise_scale;
  m.vocab = p.vocab;
  m.layers = p.layers;
  m.order = p.order;
  m.eos = p.vocab - 1;
  return m;
}

void ensure_device(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    throw Fail{FASER_ECUDA, std::string("no CUDA device available: ") + cudaGetErrorString(e)};
  if (device < 0 || device >= n) throw Fail{FASER_EINVAL, "device index out of range"};
  CK(cudaSetDevice(device));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) : n(count) {
    if (count) CK(cudaMalloc(&p, sizeof(T) * count));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct SlotBufs {
  DevBuf<int32_t> tok, len, ncomm, max_out, done, exempt, draft, draft_len;
  DevBuf<uint64_t> nh, mh, mh_at;
  SlotState view(int max_seq) const {
    SlotState s{};
    s.tok = tok.p;
    s.len = len.p;
    s.ncomm = ncomm.p;
    s.max_out = max_out.p;
    s.done = done.p;
    s.exempt = exempt.p;
    s.nh = nh.p;
    s.mh = mh.p;
    s.draft = draft.p;
    s.draft_len = draft_len.p;
    s.mh_at = mh_at.p;
    s.max_seq = max_seq;
    return s;
  }
  void alloc(int slots, int max_seq) {
    tok = DevBuf<int32_t>(static_cast<size_t>(slots) * max_seq);
    len = DevBuf<int32_t>(slots);
    ncomm = DevBuf<int32_t>(slots);
    max_out = DevBuf<int32_t>(slots);
    done = DevBuf<int32_t>(slots);
    exempt = DevBuf<int32_t>(slots);
    draft = DevBuf<int32_t>(static_cast<size_t>(slots) * FASER_MAX_SPEC);
    draft_len = DevBuf<int32_t>(slots);
    nh = DevBuf<uint64_t>(slots);
    mh = DevBuf<uint64_t>(slots);
    mh_at = DevBuf<uint64_t>(static_cast<size_t>(slots) * (FASER_MAX_SPEC + 1));
  }
};

template <class F>
faser_status guarded(std::string* err, F&& f) {
  try {
    f();
    return FASER_OK;
  } catch (const Fail& e) {
    if (err) *err = e.msg;
    g_last_error = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    if (err) *err = "host allocation failed";
    g_last_error = "host allocation failed";
    return FASER_ENOMEM;
  }
}

}  // namespace
}  // namespace faser

using namespace faser;

// ------------------------------------------------------------------------------ engine
struct faser_engine {
  faser::LlamaEngine* llama = nullptr;  // model kind LLAMA: the transformer path
  faser_engine_cfg cfg{};
  faser_toy_params toy{};
  ToyDev m{};
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  SlotBufs slots;
  StepIn* h_in = nullptr;  // pinned
  StepIn* d_in = nullptr;
  faser_round_result* h_res = nullptr;  // pinned
  double prof_pre = 0, prof_sync = 0, prof_post = 0;  // host ms per phase of faser_step (FASER_TOY_PROF)
  double prof_dev_draft = 0, prof_dev_verify = 0;      // device ms (events) of the same steps
  faser_round_result* d_res = nullptr;
  std::string err;
  int64_t launches = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  float t_draft = 0.f, t_verify = 0.f, t_step = 0.f;
  bool t_pending = false;
  const bool prof_on = std::getenv("FASER_TOY_PROF") != nullptr;
  void resolve_timing() {
    if (!t_pending) return;
    cudaEventElapsedTime(&t_draft, ev[0], ev[1]);
    cudaEventElapsedTime(&t_verify, ev[1], ev[2]);
    cudaEventElapsedTime(&t_step, ev[0], ev[2]);
    t_pending = false;
  }

  struct Req {
    int64_t id;
    std::vector<int32_t> committed;
    int32_t max_out = 0;
    int32_t prompt_len = 0;
    int32_t spec_length = 0;
    int32_t slot = -1;
    bool done = false;
    bool initialized = false;  // admit kernel enqueued
    std::vector<int32_t> prompt;  // host copy until admitted (uploaded inline with that round's StepIn)
  };
  std::unordered_map<int64_t, Req> reqs;
  std::deque<int64_t> pending;
  std::vector<int64_t> live;  // batch order
  std::vector<int32_t> free_slots;

  ~faser_engine() {
    if (llama) faser::llama_engine_destroy(llama);
    if (stream) cudaStreamSynchronize(stream);
    if (h_in) cudaFreeHost(h_in);
    if (h_res) cudaFreeHost(h_res);
    if (d_in) cudaFree(d_in);
    if (d_res) cudaFree(d_res);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }

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
};

extern "C" {

const char* faser_last_error(const faser_engine* e) {
  if (e && e->llama) return faser::llama_last_error(e->llama);
  return e ? e->err.c_str() : g_last_error.c_str();
}

faser_status faser_engine_create(const faser_model_desc* model, const faser_engine_cfg* cfg,
                                 faser_engine** out) {
  if (!out) return FASER_EINVAL;
  *out = nullptr;
  faser_engine* e = nullptr;
  if (model && cfg && model->kind == FASER_MODEL_LLAMA) {
    faser_status lst = FASER_OK;
    const char* msg = "";
    faser::LlamaEngine* le = faser::llama_engine_create(model, cfg, &lst, &msg);
    if (!le) {
      g_last_error = msg;
      return lst;
    }
    e = new faser_engine();
    e->llama = le;
    e->cfg = *cfg;
    *out = e;
    return FASER_OK;
  }
  faser_status st = guarded(nullptr, [&] {
    if (!model || !cfg) throw Fail{FASER_EINVAL, "null model or cfg"};
    if (model->kind != FASER_MODEL_TOY)
      throw Fail{FASER_ECONFIG, "model kind not supported by this engine build"};
    std::string why;
    if (!valid_toy(&model->toy, &why)) throw Fail{FASER_EINVAL, why};
    if (cfg->max_batch < 1 || cfg->max_batch > kMaxBatchHW)
      throw Fail{FASER_EINVAL, "max_batch out of range [1, 1024]"};
    if (cfg->max_seq_len < 2) throw Fail{FASER_EINVAL, "max_seq_len must be >= 2"};
    if (cfg->mode < FASER_MODE_VSD || cfg->mode > FASER_MODE_FULL)
      throw Fail{FASER_EINVAL, "unknown mode"};
    if (cfg->exempt_rule != 0 && cfg->exempt_rule != 1)
      throw Fail{FASER_EINVAL, "the toy engine follows the reference's rules: exempt_rule 0 or 1"};
    const faser_exit_policy& p = cfg->exit_policy;
    if (p.k_init < 1 || p.k_final < 1 || p.k_final > p.k_init)
      throw Fail{FASER_EINVAL, "exit policy thresholds must satisfy k_init >= k_final >= 1"};
    if (cfg->default_spec_length < 1 || cfg->default_spec_length > FASER_MAX_SPEC)
      throw Fail{FASER_EINVAL, "default_spec_length out of range"};
    ensure_device(cfg->device);
    e = new faser_engine();
    e->cfg = *cfg;
    e->toy = model->toy;
    e->m = make_toy(model->toy);
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    for (auto& ev : e->ev) CK(cudaEventCreate(&ev));
    // slot rows hold prompt ++ committed plus one round of speculative headroom
    const int row = cfg->max_seq_len + FASER_MAX_SPEC + 2;
    e->slots.alloc(cfg->max_batch, row);
    const size_t in_cap = StepIn::capacity(cfg->max_batch, static_cast<int64_t>(cfg->max_batch) * cfg->max_seq_len);
    CK(cudaMallocHost(reinterpret_cast<void**>(&e->h_in), in_cap));
    CK(cudaMalloc(reinterpret_cast<void**>(&e->d_in), in_cap));
    CK(cudaMallocHost(&e->h_res, sizeof(faser_round_result) * cfg->max_batch));
    CK(cudaMalloc(&e->d_res, sizeof(faser_round_result) * cfg->max_batch));
    std::memset(e->h_in, 0, in_cap);
    for (int s = cfg->max_batch - 1; s >= 0; --s) e->free_slots.push_back(s);
  });
  if (st != FASER_OK) {
    delete e;
    return st;
  }
  *out = e;
  return FASER_OK;
}

void faser_engine_destroy(faser_engine* e) { delete e; }

faser_status faser_submit(faser_engine* e, int64_t req_id, const int32_t* prompt, int32_t len,
                          int32_t max_out) {
  if (!e) return FASER_EINVAL;
  if (e->llama) return faser::llama_submit(e->llama, req_id, prompt, len, max_out);
  return guarded(&e->err, [&] {
    if (!prompt || len < 1) throw Fail{FASER_EINVAL, "prompt must be non-empty"};
    if (max_out < 0) throw Fail{FASER_EINVAL, "max_out must be >= 0"};
    if (e->reqs.count(req_id)) throw Fail{FASER_EINVAL, "duplicate request id"};
    if (static_cast<int64_t>(len) + max_out > e->cfg.max_seq_len)
      throw Fail{FASER_ECAPACITY, "prompt + max_out exceeds max_seq_len"};
    for (int i = 0; i < len; ++i)
      if (prompt[i] < 0 || prompt[i] >= e->toy.vocab) throw Fail{FASER_EINVAL, "token outside vocabulary"};
    faser_engine::Req r;
    r.id = req_id;
    r.max_out = max_out;
    r.prompt_len = len;
    r.spec_length = e->cfg.default_spec_length;
    r.done = max_out == 0;  // Request::done invariant: |committed| == max_out
    if (!r.done) r.prompt.assign(prompt, prompt + len);
    r.committed.reserve(max_out);
    e->reqs.emplace(req_id, std::move(r));
    if (max_out > 0) e->pending.push_back(req_id);
  });
}

faser_status faser_set_spec_lengths(faser_engine* e, const int64_t* req_ids, const int32_t* k,
                                    int32_t n) {
  if (!e) return FASER_EINVAL;
  if (e->llama) return faser::llama_set_spec_lengths(e->llama, req_ids, k, n);
  return guarded(&e->err, [&] {
    for (int i = 0; i < n; ++i) {
      if (k[i] < 1 || k[i] > FASER_MAX_SPEC)
        throw Fail{FASER_EINVAL, "speculative length must be in [1, FASER_MAX_SPEC]"};
      auto it = e->reqs.find(req_ids[i]);
      if (it == e->reqs.end()) throw Fail{FASER_EINVAL, "unknown request id"};
      it->second.spec_length = k[i];
    }
  });
}

faser_status faser_live_requests(faser_engine* e, int64_t* req_ids, int32_t cap, int32_t* n) {
  if (!e || !n) return FASER_EINVAL;
  if (e->llama) return faser::llama_live_requests(e->llama, req_ids, cap, n);
  return guarded(&e->err, [&] {
    e->admit_pending();
    *n = static_cast<int32_t>(e->live.size());
    for (int i = 0; i < *n && i < cap; ++i) req_ids[i] = e->live[i];
  });
}

int32_t faser_pending_work(const faser_engine* e) {
  if (e && e->llama) return faser::llama_pending_work(e->llama);
  return e ? static_cast<int32_t>(e->live.size() + e->pending.size()) : 0;
}

faser_status faser_step(faser_engine* e, const faser_step_plan* plan, faser_round_result* out,
                        int32_t cap, int32_t* n_out) {
  if (!e || !n_out) return FASER_EINVAL;
  if (e->llama) return faser::llama_step(e->llama, plan, out, cap, n_out);
  return guarded(&e->err, [&] {
    const auto q0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(e->cfg.device));
    e->admit_pending();
    const int n_live = static_cast<int>(e->live.size());
    *n_out = n_live;
    if (n_live == 0) return;
    if (cap < n_live) throw Fail{FASER_ECAPACITY, "result capacity smaller than live batch"};
    StepIn& in = *e->h_in;
    const int L = e->toy.layers;
    int n_admit = 0, n_ptok = 0;
    for (int p = 0; p < n_live; ++p) {
      const faser_engine::Req& r = e->reqs.at(e->live[p]);
      if (!r.initialized) {
        ++n_admit;
        n_ptok += r.prompt_len;
      }
    }
    in.layout(n_live, n_admit, n_ptok);
    in.early_exit = e->cfg.mode >= FASER_MODE_VSD_AD_EE ? 1 : 0;
    in.commit = 1;
    in.exempt_rule = e->cfg.exempt_rule;
    faser_gate_plan g{e->cfg.exit_policy.l_init, e->cfg.exit_policy.l_init, 1.0};
    if (plan) g = plan->gate;
    in.gate_lo = std::max(g.first_layer, 1);
    in.gate_hi = std::min(g.stop_layer, L);
    if (!(g.first_layer < g.stop_layer)) in.gate_lo = in.gate_hi = 0;  // GatePlan::active()
    if (plan && plan->use_k_table) {
      for (int l = 0; l <= L; ++l) {
        if (plan->k_table[l] < 1) throw Fail{FASER_EINVAL, "k must be >= 1"};
        in.k_table[l] = plan->k_table[l];
      }
    } else if (faser_k_table(&e->cfg.exit_policy, L, in.k_table) != FASER_OK) {
      throw Fail{FASER_EINVAL, "invalid exit policy"};
    }
    int ai = 0, toff = 0;
    const int32_t* d_tok = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(e->d_in) + in.off_tok);
    for (int p = 0; p < n_live; ++p) {
      faser_engine::Req& r = e->reqs.at(e->live[p]);
      in.live_slot()[p] = r.slot;
      in.k()[p] = r.spec_length;
      in.req_id()[p] = r.id;
      if (!r.initialized) {
        AdmitEntry& a = in.admit()[ai++];
        std::memcpy(in.tok() + toff, r.prompt.data(), sizeof(int32_t) * r.prompt_len);
        a.src = d_tok + toff;
        toff += r.prompt_len;
        std::vector<int32_t>().swap(r.prompt);
        r.initialized = true;
        a.slot = r.slot;
        a.len = r.prompt_len;
        a.max_out = r.max_out;
        a.ncomm = 0;
        a.exempt = -1;
      }
    }
    CK(cudaMemcpyAsync(e->d_in, e->h_in, in.total_bytes, cudaMemcpyHostToDevice, e->stream));
    e->h2d_bytes = in.total_bytes;
    e->d2h_bytes = static_cast<int64_t>(sizeof(faser_round_result)) * n_live;
    SlotState sv = e->slots.view(e->cfg.max_seq_len + FASER_MAX_SPEC + 2);
    CK(cudaEventRecord(e->ev[0], e->stream));
    // admission + draft + verify + commit fused per request (one launch; t_draft = 0)
    CK(cudaEventRecord(e->ev[1], e->stream));
    CK(toy_draft_verify_commit(e->m, sv, e->d_in, n_live, e->d_res, e->stream));
    CK(cudaEventRecord(e->ev[2], e->stream));
    e->launches += 1;
    CK(cudaMemcpyAsync(e->h_res, e->d_res, sizeof(faser_round_result) * n_live,
                       cudaMemcpyDeviceToHost, e->stream));
    const auto q1 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(e->stream));
    const auto q2 = std::chrono::steady_clock::now();
    e->t_pending = true;  // resolved on demand (faser_last_step_timing): three driver calls per round
    if (e->prof_on) e->resolve_timing();
    std::vector<int64_t> keep;
    keep.reserve(n_live);
    for (int p = 0; p < n_live; ++p) {
      const faser_round_result& rr = e->h_res[p];
      faser_engine::Req& r = e->reqs.at(e->live[p]);
      r.committed.insert(r.committed.end(), rr.tokens, rr.tokens + rr.committed);
      r.done = rr.done != 0;
      if (r.done) {
        e->free_slots.push_back(r.slot);
        r.slot = -1;
      } else {
        keep.push_back(r.id);
      }
    }
    std::memcpy(out, e->h_res, sizeof(faser_round_result) * n_live);
    e->live.swap(keep);
    const auto q3 = std::chrono::steady_clock::now();
    e->prof_pre += std::chrono::duration<double, std::milli>(q1 - q0).count();
    e->prof_sync += std::chrono::duration<double, std::milli>(q2 - q1).count();
    e->prof_post += std::chrono::duration<double, std::milli>(q3 - q2).count();
    e->prof_dev_draft += e->t_draft;
    e->prof_dev_verify += e->t_verify;
  });
}

faser_status faser_get_committed(faser_engine* e, int64_t req_id, int32_t* buf, int32_t cap,
                                 int32_t* n) {
  if (!e || !n) return FASER_EINVAL;
  if (e->llama) return faser::llama_get_committed(e->llama, req_id, buf, cap, n);
  return guarded(&e->err, [&] {
    auto it = e->reqs.find(req_id);
    if (it == e->reqs.end()) throw Fail{FASER_EINVAL, "unknown request id"};
    const auto& c = it->second.committed;
    *n = static_cast<int32_t>(c.size());
    if (buf) std::memcpy(buf, c.data(), sizeof(int32_t) * std::min<size_t>(c.size(), std::max(cap, 0)));
  });
}

faser_status faser_release(faser_engine* e, int64_t req_id) {
  if (!e) return FASER_EINVAL;
  if (e->llama) return faser::llama_release(e->llama, req_id);
  return guarded(&e->err, [&] {
    auto it = e->reqs.find(req_id);
    if (it == e->reqs.end()) throw Fail{FASER_EINVAL, "unknown request id"};
    if (!it->second.done) throw Fail{FASER_EILLEGAL_STATE, "release of a live request"};
    e->reqs.erase(it);
  });
}

faser_status faser_debug_set_skip_mask(faser_engine* e, int32_t mask) {
  if (!e || !e->llama) return FASER_EINVAL;
  return faser::llama_set_skip_mask(e->llama, mask);
}

faser_status faser_set_sampling(faser_engine* e, double temperature, uint64_t seed) {
  if (!e || !e->llama) return FASER_EINVAL;
  return faser::llama_set_sampling(e->llama, temperature, seed);
}

faser_status faser_set_prefill_lane(faser_engine* e, int32_t on) {
  if (!e) return FASER_EINVAL;
  if (!e->llama) return on ? FASER_EINVAL : FASER_OK;
  return faser::llama_set_prefill_lane(e->llama, on);
}

faser_status faser_engine_join_lanes(faser_engine* e) {
  if (!e) return FASER_EINVAL;
  return e->llama ? faser::llama_join_lanes(e->llama) : FASER_OK;
}

faser_status faser_last_step_prefill(const faser_engine* e, float* prefill_ms) {
  if (!e || !prefill_ms) return FASER_EINVAL;
  *prefill_ms = e->llama ? faser::llama_last_step_prefill(e->llama) : 0.f;
  return FASER_OK;
}

faser_status faser_last_step_timing(const faser_engine* e, float* draft_ms, float* verify_ms,
                                    float* step_ms) {
  if (!e) return FASER_EINVAL;
  if (e->llama) {
    faser::llama_last_step_timing(e->llama, draft_ms, verify_ms, step_ms);
    return FASER_OK;
  }
  const_cast<faser_engine*>(e)->resolve_timing();
  if (draft_ms) *draft_ms = e->t_draft;
  if (verify_ms) *verify_ms = e->t_verify;
  if (step_ms) *step_ms = e->t_step;
  return FASER_OK;
}

int64_t faser_kernel_launches(const faser_engine* e) {
  if (e && e->llama) return faser::llama_launches(e->llama);
  return e ? e->launches : 0;
}

faser_status faser_last_step_bytes(const faser_engine* e, int64_t* h2d, int64_t* d2h) {
  if (!e) return FASER_EINVAL;
  if (e->llama) {
    faser::llama_last_step_bytes(e->llama, h2d, d2h);
    return FASER_OK;
  }
  if (h2d) *h2d = e->h2d_bytes;
  if (d2h) *d2h = e->d2h_bytes;
  return FASER_OK;
}

faser_status faser_last_timeline(const faser_engine* e, faser_timeline_event* ev, int32_t cap,
                                 faser_timeline_info* info) {
  if (!e || !info || cap < 0 || (cap > 0 && !ev)) return FASER_EINVAL;
  if (!e->llama) return FASER_EINVAL;  // the toy engine runs its rounds serially
  return faser::llama_last_timeline(e->llama, ev, cap, info);
}

void* faser_engine_stream(const faser_engine* e) {
  if (e && e->llama) return faser::llama_stream(e->llama);
  return e ? static_cast<void*>(e->stream) : nullptr;
}

faser_status faser_debug_verify_logits(faser_engine* e, int32_t stage, float* logits, int64_t* row_ids,
                                       int32_t cap_rows, int32_t* rows) {
  if (!e || !rows) return FASER_EINVAL;
  if (!e->llama) return FASER_EINVAL;
  return faser::llama_debug_verify_logits(e->llama, stage, logits, row_ids, cap_rows, rows);
}

faser_status faser_debug_drafted(faser_engine* e, int32_t* drafted, int32_t cap, int32_t* n) {
  if (!e || !n || !e->llama) return FASER_EINVAL;
  return faser::llama_debug_drafted(e->llama, drafted, cap, n);
}

faser_status faser_debug_weights(faser_engine* e, int32_t model, int32_t which, int32_t layer,
                                 int64_t offset, int32_t n, uint16_t* out) {
  if (!e || !e->llama) return FASER_EINVAL;
  return faser::llama_debug_weights(e->llama, model, which, layer, offset, n, out);
}

faser_status faser_set_kernel_timing(faser_engine* e, int32_t enabled) {
  if (!e || !e->llama) return FASER_EINVAL;
  return faser::llama_set_kernel_timing(e->llama, enabled);
}

faser_status faser_kernel_stats(faser_engine* e, int32_t cls, double* ms, int64_t* launches, double* bytes) {
  if (!e || !e->llama) return FASER_EINVAL;
  return faser::llama_kernel_stats(e->llama, cls, ms, launches, bytes);
}

faser_status faser_kernel_flops(faser_engine* e, int32_t cls, double* flops) {
  if (!e || !e->llama) return FASER_EINVAL;
  return faser::llama_kernel_flops(e->llama, cls, flops);
}

faser_status faser_debug_kv_pages(faser_engine* e, int64_t req_id, int32_t* pages, int32_t cap, int32_t* n) {
  if (!e || !n || !e->llama) return FASER_EINVAL;
  return faser::llama_debug_kv_pages(e->llama, req_id, pages, cap, n);
}

// --------------------------------------------------------------- stateless batched toy ops

namespace {

struct Ragged {
  DevBuf<int32_t> tok;
  DevBuf<int64_t> off;
};

void validate_ragged(int n, const int32_t* tokens, const int64_t* offsets, int vocab) {
  if (n < 0 || (n > 0 && (!tokens || !offsets))) throw Fail{FASER_EINVAL, "null ragged batch"};
  for (int i = 0; i < n; ++i)
    if (offsets[i + 1] <= offsets[i]) throw Fail{FASER_EINVAL, "prefix must be non-empty"};
  const int64_t total = n ? offsets[n] - offsets[0] : 0;
  for (int64_t i = 0; i < total; ++i)
    if (tokens[offsets[0] + i] < 0 || tokens[offsets[0] + i] >= vocab)
      throw Fail{FASER_EINVAL, "token outside vocabulary"};
}

Ragged upload_ragged(int n, const int32_t* tokens, const int64_t* offsets, cudaStream_t s,
                     int vocab) {
  validate_ragged(n, tokens, offsets, vocab);
  const int64_t total = n ? offsets[n] - offsets[0] : 0;
  Ragged r;
  r.tok = DevBuf<int32_t>(std::max<int64_t>(total, 1));
  r.off = DevBuf<int64_t>(n + 1);
  std::vector<int64_t> rel(n + 1);
  for (int i = 0; i <= n; ++i) rel[i] = offsets[i] - offsets[0];
  if (total) CK(cudaMemcpyAsync(r.tok.p, tokens + offsets[0], sizeof(int32_t) * total, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(r.off.p, rel.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  return r;
}

faser_status rows_op(const faser_toy_params* model, int op, int32_t n, const int32_t* tokens,
                     const int64_t* offsets, const int32_t* layers, double* z0, double* z1,
                     int32_t* out) {
  return guarded(nullptr, [&] {
    std::string why;
    if (!valid_toy(model, &why)) throw Fail{FASER_EINVAL, why};
    if (op == 1)
      for (int i = 0; i < n; ++i)
        if (layers[i] < 1 || layers[i] > model->layers)
          throw Fail{FASER_EINVAL, "layer out of range [1, layers]"};
    validate_ragged(n, tokens, offsets, model->vocab);
    ensure_device(0);
    const ToyDev m = make_toy(*model);
    cudaStream_t s = nullptr;
    Ragged r = upload_ragged(n, tokens, offsets, s, model->vocab);
    DevBuf<int32_t> d_layers(op == 1 ? n : 0), d_out(op >= 2 ? n : 0);
    DevBuf<double> d_z0(op <= 1 ? static_cast<size_t>(n) * model->vocab : 0),
        d_z1(op == 0 ? static_cast<size_t>(n) * model->vocab : 0);
    if (op == 1) CK(cudaMemcpyAsync(d_layers.p, layers, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CK(toy_rows(m, op, n, r.tok.p, r.off.p, d_layers.p, d_z0.p, d_z1.p, d_out.p, s));
    if (op <= 1) CK(cudaMemcpyAsync(z0, d_z0.p, sizeof(double) * n * model->vocab, cudaMemcpyDeviceToHost, s));
    if (op == 0) CK(cudaMemcpyAsync(z1, d_z1.p, sizeof(double) * n * model->vocab, cudaMemcpyDeviceToHost, s));
    if (op >= 2) CK(cudaMemcpyAsync(out, d_out.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

}  // namespace

faser_status faser_toy_final_and_noise(const faser_toy_params* model, int32_t n,
                                       const int32_t* tokens, const int64_t* offsets,
                                       double* z_final, double* z_noise) {
  return rows_op(model, 0, n, tokens, offsets, nullptr, z_final, z_noise, nullptr);
}

faser_status faser_toy_target_logits(const faser_toy_params* model, int32_t n,
                                     const int32_t* tokens, const int64_t* offsets,
                                     const int32_t* layers, double* z) {
  if (!layers && n > 0) return FASER_EINVAL;
  return rows_op(model, 1, n, tokens, offsets, layers, z, nullptr, nullptr);
}

faser_status faser_toy_target_next(const faser_toy_params* model, int32_t n,
                                   const int32_t* tokens, const int64_t* offsets, int32_t* out) {
  return rows_op(model, 2, n, tokens, offsets, nullptr, nullptr, nullptr, out);
}

faser_status faser_toy_draft_next(const faser_toy_params* model, int32_t n,
                                  const int32_t* tokens, const int64_t* offsets, int32_t* out) {
  return rows_op(model, 3, n, tokens, offsets, nullptr, nullptr, nullptr, out);
}

// Shared by faser_toy_draft_tokens / faser_toy_verify: materialise a temporary slot table
// from the ragged contexts (admit kernel), then run the same draft / verify kernels the
// engine runs, with commit disabled.
static void run_stateless(const faser_toy_params* model, int32_t n, const int32_t* tokens,
                          const int64_t* offsets, const int32_t* committed_len,
                          const int32_t* exempt, const int32_t* s, const int32_t* remaining,
                          const int32_t* drafted, const int32_t* drafted_len,
                          const faser_exit_policy* policy, const faser_gate_plan* gate,
                          int32_t* out_tokens, int32_t* out_len, faser_verify_outcome* outcomes) {
  std::string why;
  if (!valid_toy(model, &why)) throw Fail{FASER_EINVAL, why};
  if (n < 0 || n > kMaxBatchHW) throw Fail{FASER_EINVAL, "batch size out of range [0, 1024]"};
  if (n == 0) return;
  ensure_device(0);
  const bool verify = drafted != nullptr;
  if (verify && gate) {
    if (!policy || policy->k_init < 1 || policy->k_final < 1 || policy->k_final > policy->k_init)
      throw Fail{FASER_EINVAL, "exit policy thresholds must satisfy k_init >= k_final >= 1"};
  }
  const ToyDev m = make_toy(*model);
  cudaStream_t st = nullptr;
  Ragged r = upload_ragged(n, tokens, offsets, st, model->vocab);
  int64_t maxlen = 0;
  for (int i = 0; i < n; ++i) maxlen = std::max<int64_t>(maxlen, offsets[i + 1] - offsets[i]);
  const int max_seq = static_cast<int>(maxlen) + FASER_MAX_SPEC + 2;
  SlotBufs b;
  b.alloc(n, max_seq);
  std::vector<uint64_t> hin_buf(StepIn::capacity(n) / 8 + 1, 0);
  StepIn& in = *reinterpret_cast<StepIn*>(hin_buf.data());
  in.layout(n, n);
  in.commit = 0;
  in.early_exit = (verify && gate) ? 1 : 0;
  if (in.early_exit) {
    in.gate_lo = std::max(gate->first_layer, 1);
    in.gate_hi = std::min(gate->stop_layer, model->layers);
    if (!(gate->first_layer < gate->stop_layer)) in.gate_lo = in.gate_hi = 0;
    if (faser_k_table(policy, model->layers, in.k_table) != FASER_OK)
      throw Fail{FASER_EINVAL, "invalid exit policy"};
  }
  std::vector<int32_t> dl(n), dtok(static_cast<size_t>(n) * FASER_MAX_SPEC, 0);
  for (int i = 0; i < n; ++i) {
    const int len = static_cast<int>(offsets[i + 1] - offsets[i]);
    AdmitEntry& a = in.admit()[i];
    a.src = r.tok.p + (offsets[i] - offsets[0]);
    a.slot = i;
    a.len = len;
    in.live_slot()[i] = i;
    in.req_id()[i] = i;
    if (verify) {
      const int c = drafted_len[i];
      if (c < 1) throw Fail{FASER_EINVAL, "verify on empty draft"};
      if (c > FASER_MAX_SPEC) throw Fail{FASER_EINVAL, "draft longer than FASER_MAX_SPEC"};
      const int cl = committed_len ? committed_len[i] : 0;
      if (cl < 0 || cl > len) throw Fail{FASER_EINVAL, "committed_len outside context"};
      for (int j = 0; j < c; ++j) {
        const int32_t t = drafted[static_cast<int64_t>(i) * FASER_MAX_SPEC + j];
        if (t < 0 || t >= model->vocab) throw Fail{FASER_EINVAL, "drafted token outside vocabulary"};
        dtok[static_cast<size_t>(i) * FASER_MAX_SPEC + j] = t;
      }
      dl[i] = c;
      a.ncomm = cl;
      a.max_out = cl + FASER_MAX_SPEC + 1;
      a.exempt = exempt ? exempt[i] : -1;
      in.k()[i] = c;
    } else {
      if (remaining[i] <= 0) throw Fail{FASER_EILLEGAL_STATE, "draft_tokens on a finished request"};
      if (s[i] < 1) throw Fail{FASER_EINVAL, "speculative length must be >= 1"};
      if (s[i] > FASER_MAX_SPEC) throw Fail{FASER_EINVAL, "speculative length > FASER_MAX_SPEC"};
      a.ncomm = 0;
      a.max_out = remaining[i];
      a.exempt = -1;
      in.k()[i] = s[i];
    }
  }
  DevBuf<uint64_t> d_in_buf(hin_buf.size());
  const StepIn* d_in = reinterpret_cast<const StepIn*>(d_in_buf.p);
  DevBuf<faser_round_result> d_res(verify ? n : 0);
  CK(cudaMemcpyAsync(d_in_buf.p, &in, in.total_bytes, cudaMemcpyHostToDevice, st));
  SlotState sv = b.view(max_seq);
  CK(toy_admit(m, sv, d_in, n, st));
  if (verify) {
    CK(cudaMemcpyAsync(b.draft.p, dtok.data(), sizeof(int32_t) * dtok.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(b.draft_len.p, dl.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    CK(toy_verify_commit(m, sv, d_in, n, d_res.p, st));
    std::vector<faser_round_result> res(n);
    CK(cudaMemcpyAsync(res.data(), d_res.p, sizeof(faser_round_result) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int i = 0; i < n; ++i) outcomes[i] = res[i].outcome;
  } else {
    CK(toy_draft(m, sv, d_in, n, st));
    CK(cudaMemcpyAsync(out_tokens, b.draft.p, sizeof(int32_t) * n * FASER_MAX_SPEC, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_len, b.draft_len.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
}

faser_status faser_toy_draft_tokens(const faser_toy_params* model, int32_t n,
                                    const int32_t* tokens, const int64_t* offsets,
                                    const int32_t* s, const int32_t* remaining,
                                    int32_t* out, int32_t* out_len) {
  if (n > 0 && (!s || !remaining || !out || !out_len)) return FASER_EINVAL;
  return guarded(nullptr, [&] {
    run_stateless(model, n, tokens, offsets, nullptr, nullptr, s, remaining, nullptr, nullptr,
                  nullptr, nullptr, out, out_len, nullptr);
  });
}

faser_status faser_toy_verify(const faser_toy_params* model, int32_t n, const int32_t* tokens,
                              const int64_t* offsets, const int32_t* committed_len,
                              const int32_t* exempt, const int32_t* drafted,
                              const int32_t* drafted_len, const faser_exit_policy* policy,
                              const faser_gate_plan* gate, faser_verify_outcome* out) {
  if (n > 0 && (!drafted || !drafted_len || !out)) return FASER_EINVAL;
  return guarded(nullptr, [&] {
    run_stateless(model, n, tokens, offsets, committed_len, exempt, nullptr, nullptr, drafted,
                  drafted_len, policy, gate, nullptr, nullptr, out);
  });
}

}  // extern "C"

// ------------------------------------------------------------------ serving loop (sim.cpp role)
namespace {
constexpr uint64_t kSrvGamma = 0x9e3779b97f4a7c15ull;
uint64_t srv_mix64(uint64_t x) {  // rng.hpp:17-22
  x += kSrvGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t srv_hash_combine(uint64_t h, uint64_t v) {  // rng.hpp:24-26
  return srv_mix64(h ^ (v + kSrvGamma + (h << 6) + (h >> 2)));
}
constexpr int32_t kSrvCandidates[8] = {1, 2, 3, 4, 5, 6, 8, 10};  // drafter.hpp:16
}  // namespace

extern "C" faser_status faser_serve_rounds(faser_engine* e, int32_t n_rounds, uint64_t seed, int64_t id_base,
                                           const faser_exit_policy* policy, double accept_est, double r,
                                           int32_t num_layers, int64_t* tokens_out, int32_t* rounds_out) {
  if (!e || n_rounds < 0 || !tokens_out || !rounds_out) return FASER_EINVAL;
  *tokens_out = 0;
  *rounds_out = 0;
  const int cap = 1 << 12;
  std::vector<int64_t> ids(cap);
  std::vector<int32_t> ks(cap);
  std::vector<faser_gate_entry> ents(cap);
  std::vector<faser_round_result> res(cap);
  std::unordered_map<int64_t, int32_t> served;
  // FASER_TOY_PROF=1: host time per phase of the loop, printed at the end (stderr)
  static const bool prof = std::getenv("FASER_TOY_PROF") != nullptr;
  using clk = std::chrono::steady_clock;
  double t_live = 0, t_k = 0, t_gate = 0, t_step = 0, t_post = 0;
  auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  for (int it = 0; it < n_rounds; ++it) {
    const auto p0 = clk::now();
    int32_t n = 0;
    faser_status st = faser_live_requests(e, ids.data(), cap, &n);
    if (st != FASER_OK) return st;
    if (n == 0) break;
    if (n > cap) return FASER_ECAPACITY;
    const auto p1 = clk::now();
    for (int i = 0; i < n; ++i) {
      const int32_t rnd = served[ids[i]];
      const uint64_t h = srv_hash_combine(srv_hash_combine(srv_mix64(seed), static_cast<uint64_t>(ids[i] - id_base + 1)),
                                          static_cast<uint64_t>(rnd + 1));
      ks[i] = kSrvCandidates[h % 8];
    }
    if ((st = faser_set_spec_lengths(e, ids.data(), ks.data(), n)) != FASER_OK) return st;
    const auto p2 = clk::now();
    faser_step_plan plan{};
    if (policy) {
      for (int i = 0; i < n; ++i) {
        ents[i] = faser_gate_entry{};
        ents[i].spec_length = ks[i];
        ents[i].accept_estimate = accept_est;
      }
      if ((st = faser_make_gate_plan(policy, ents.data(), n, static_cast<double>(n), r, nullptr, num_layers,
                                     &plan.gate)) != FASER_OK)
        return st;
    }
    const auto p3 = clk::now();
    int32_t got = 0;
    if ((st = faser_step(e, policy ? &plan : nullptr, res.data(), cap, &got)) != FASER_OK) return st;
    const auto p4 = clk::now();
    for (int i = 0; i < got; ++i) {
      served[res[i].req_id] += 1;
      *tokens_out += res[i].committed;
    }
    if (prof) {
      const auto p5 = clk::now();
      t_live += ms(p0, p1);
      t_k += ms(p1, p2);
      t_gate += ms(p2, p3);
      t_step += ms(p3, p4);
      t_post += ms(p4, p5);
    }
    *rounds_out += 1;
  }
  if (prof && *rounds_out > 0) {
    const double n = *rounds_out;
    std::fprintf(stderr, "serve_rounds host ms/round: live %.4f k %.4f gate %.4f step %.4f (pre-launch %.4f, sync wait %.4f, post %.4f) loop-post %.4f; device admit+draft %.4f verify %.4f\n",
                 t_live / n, t_k / n, t_gate / n, t_step / n, e->prof_pre / n, e->prof_sync / n, e->prof_post / n, t_post / n,
                 e->prof_dev_draft / n, e->prof_dev_verify / n);
    e->prof_pre = e->prof_sync = e->prof_post = e->prof_dev_draft = e->prof_dev_verify = 0;
  }
  return FASER_OK;
}

// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Builds `oracle/_ref/libspecsim_ref.so` from the reference's OWN translation units,
// compiled in place from /root/reference/proj/core/src/{toylm,sdcore,exitctl,overlap,
// workload}.cpp (see oracle/Makefile). This file adds:
//   1. the one symbol those TUs need that lives in an unbuildable TU (latmodel.cpp needs
//      Eigen, absent on this image): eval_latency + default_ground_truth, restated from
//      latmodel.cpp:32-62 and latmodel.cpp:396-403;
//   2. extern "C" wrappers over the reference classes, using the product's public structs
//      (include/faser/engine.h) so tests compare records field by field;
//   3. a serving-loop episode runner over the reference SpeculativeEngine (the reference's
//      sim.cpp is absent; the loop follows SPEC.md:541-563 and SURVEY.md §3(A)), threaded
//      with a persistent pool: this is the reference CPU baseline timed by bench.py.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load this library.

#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <thread>
#include <vector>

#include "faser/engine.h"
#include "oracle.h"
#include "specsim/exitctl.hpp"
#include "specsim/drafter.hpp"
#include "specsim/latmodel.hpp"
#ifdef SPECREF_METRICS
#include "specsim/metrics.hpp"
#endif
#include "specsim/overlap.hpp"
#include "specsim/rng.hpp"
#include "specsim/sdcore.hpp"
#include "specsim/toylm.hpp"
#include "specsim/workload.hpp"

namespace specsim {
// ---- restated from latmodel.cpp (Eigen-free part only) ----
double own_share(StageKind stage, double r) {
  return (stage == StageKind::Draft || stage == StageKind::Prune) ? r : 1.0 - r;
}
double piecewise_factor(const PiecewiseLatencyParams& p, double x) {
  if (!(x > 0.0) || x > 1.0) throw std::invalid_argument("SM share outside (0,1]");
  return x <= p.knee ? p.a1 - p.gamma1 * x : p.a2 - p.gamma2 * x;
}
double load_term(const PiecewiseLatencyParams& p, double b, double s) {
  switch (p.stage) {
    case StageKind::Draft: return p.c0 * b + p.c1 * s + p.c2;
    case StageKind::Target: return (p.c0 * b + p.c1) * s + p.c2;
    default: return p.c0 * b * s + p.c1;
  }
}
double eval_latency(const PiecewiseLatencyParams& p, double b, double s, double r) {
  return piecewise_factor(p, own_share(p.stage, r)) * load_term(p, b, s);
}
LatencyModel LatencyModel::default_ground_truth() {
  LatencyModel m;
  m.draft = {StageKind::Draft, 0.5, 1.6, 0.9, 1.275, 0.25, 0.003, 0.28, 0.5};
  m.target = {StageKind::Target, 0.5, 1.5, 0.8, 1.2, 0.2, 0.008, 0.18, 0.3};
  m.ee_check = {StageKind::EarlyExitCheck, 0.5, 1.6, 1.0, 1.3, 0.4, 2e-6, 0.002, 0.0};
  m.prune = {StageKind::Prune, 0.6, 1.5, 1.0, 1.2, 0.5, 2e-6, 0.003, 0.0};
  return m;
}
}  // namespace specsim

using namespace specsim;

namespace {

LayeredToyLM::Params to_params(const faser_toy_params* p) {
  LayeredToyLM::Params q;
  q.seed = p->seed;
  q.vocab = p->vocab;
  q.layers = p->layers;
  q.order = p->order;
  q.divergence = p->divergence;
  q.noise_seed = p->noise_seed;
  q.logit_scale = p->logit_scale;
  q.noise_scale = p->noise_scale;
  return q;
}

std::span<const int> row(const int32_t* tokens, const int64_t* off, int i) {
  return {reinterpret_cast<const int*>(tokens) + off[i], static_cast<size_t>(off[i + 1] - off[i])};
}

ExitPolicy to_policy(const faser_exit_policy* p) {
  ExitPolicy e;
  e.l_init = p->l_init;
  e.k_init = p->k_init;
  e.k_final = p->k_final;
  return e;
}

void to_c(const VerifyOutcome& o, faser_verify_outcome* out) {
  std::memset(out, 0, sizeof(*out));
  out->submitted = o.submitted;
  out->accepted_count = o.accepted_count;
  out->has_recovery = o.recovery_token.has_value();
  out->recovery_token = o.recovery_token.value_or(-1);
  out->has_pruned = o.pruned_at.has_value();
  out->pruned_index = o.pruned_at ? o.pruned_at->first : -1;
  out->pruned_layer = o.pruned_at ? o.pruned_at->second : -1;
  out->gate_layers = o.gate_layers;
  out->full_layers_run = o.full_layers_run;
  out->false_prune = o.false_prune;
  out->n_prune_layers = static_cast<int32_t>(std::min<size_t>(o.prune_layers.size(), FASER_MAX_SPEC));
  for (int i = 0; i < out->n_prune_layers; ++i) out->prune_layers[i] = o.prune_layers[i];
  out->base_len = static_cast<int64_t>(o.base_len);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return FASER_OK;
  } catch (const std::invalid_argument&) {
    return FASER_EINVAL;
  } catch (const std::logic_error&) {
    return FASER_EILLEGAL_STATE;
  } catch (...) {
    return FASER_EINVAL;
  }
}

// Sense-reversing spin barrier: rounds are ~10-300 us, so futex sleep/wake latency
// (std::barrier) would dominate; the pool owns its cores for the duration of a run.
class SpinBarrier {
 public:
  explicit SpinBarrier(int n) : n_(n) {}
  void arrive_and_wait() {
    const int gen = gen_.load(std::memory_order_acquire);
    if (count_.fetch_add(1, std::memory_order_acq_rel) + 1 == n_) {
      count_.store(0, std::memory_order_relaxed);
      gen_.fetch_add(1, std::memory_order_acq_rel);
      return;
    }
    int spins = 0;
    while (gen_.load(std::memory_order_acquire) == gen) {
      if (++spins > 4096) {
        std::this_thread::yield();
        spins = 0;
      }
    }
  }

 private:
  const int n_;
  std::atomic<int> count_{0};
  std::atomic<int> gen_{0};
};

}  // namespace

extern "C" {

int specref_final_and_noise(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                            const int64_t* off, double* zf, double* zn) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    std::vector<double> a, b;
    for (int i = 0; i < n; ++i) {
      m.final_and_noise(row(tokens, off, i), a, b);
      std::copy(a.begin(), a.end(), zf + static_cast<int64_t>(i) * p->vocab);
      std::copy(b.begin(), b.end(), zn + static_cast<int64_t>(i) * p->vocab);
    }
  });
}

int specref_target_logits(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                          const int64_t* off, const int32_t* layers, double* z) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    for (int i = 0; i < n; ++i) {
      auto v = m.target_logits(row(tokens, off, i), layers[i]);
      std::copy(v.begin(), v.end(), z + static_cast<int64_t>(i) * p->vocab);
    }
  });
}

int specref_target_next(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                        const int64_t* off, int32_t* out) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    for (int i = 0; i < n; ++i) out[i] = m.target_next(row(tokens, off, i));
  });
}

int specref_draft_next(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                       const int64_t* off, int32_t* out) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    for (int i = 0; i < n; ++i) out[i] = m.draft_next(row(tokens, off, i));
  });
}

int specref_argmax_lowest(const double* v, int32_t n, int32_t* out) {
  return guard([&] { *out = argmax_lowest({v, static_cast<size_t>(n)}); });
}

int specref_autoregressive_decode(const faser_toy_params* p, const int32_t* prompt, int32_t len,
                                  int32_t max_out, int32_t* out, int32_t* n_out) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    auto v = m.autoregressive_decode({reinterpret_cast<const int*>(prompt), static_cast<size_t>(len)},
                                     max_out);
    std::copy(v.begin(), v.end(), out);
    *n_out = static_cast<int32_t>(v.size());
  });
}

int specref_draft_tokens(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                         const int64_t* off, const int32_t* s, const int32_t* remaining,
                         int32_t* out, int32_t* out_len) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    SpeculativeEngine eng(&m);
    for (int i = 0; i < n; ++i) {
      Request req;
      auto r = row(tokens, off, i);
      req.prompt.assign(r.begin(), r.end());
      req.max_out = remaining[i];
      req.done = remaining[i] <= 0;
      auto d = eng.draft_tokens(req, s[i]);
      out_len[i] = static_cast<int32_t>(d.size());
      std::copy(d.begin(), d.end(), out + static_cast<int64_t>(i) * FASER_MAX_SPEC);
    }
  });
}

int specref_verify(const faser_toy_params* p, int32_t n, const int32_t* tokens, const int64_t* off,
                   const int32_t* committed_len, const int32_t* exempt, const int32_t* drafted,
                   const int32_t* drafted_len, const faser_exit_policy* policy,
                   const faser_gate_plan* gate, faser_verify_outcome* out) {
  return guard([&] {
    LayeredToyLM m(to_params(p));
    SpeculativeEngine eng(&m);
    for (int i = 0; i < n; ++i) {
      Request req;
      auto r = row(tokens, off, i);
      const size_t split = r.size() - static_cast<size_t>(committed_len[i]);
      req.prompt.assign(r.begin(), r.begin() + split);
      req.committed.assign(r.begin() + split, r.end());
      req.exempt_position = exempt ? exempt[i] : -1;
      std::span<const int> d(reinterpret_cast<const int*>(drafted) + static_cast<int64_t>(i) * FASER_MAX_SPEC,
                             static_cast<size_t>(drafted_len[i]));
      VerifyOutcome o;
      if (gate == nullptr) {
        o = eng.full_verify(req, d);
      } else {
        GatePlan g;
        g.first_layer = gate->first_layer;
        g.stop_layer = gate->stop_layer;
        g.s_eff = gate->s_eff;
        o = eng.verify_with_early_exit(req, d, to_policy(policy), g);
      }
      to_c(o, out + i);
    }
  });
}

int specref_k_at(const faser_exit_policy* policy, int32_t layer, int32_t num_layers, int32_t* out) {
  return guard([&] { *out = to_policy(policy).k_at(layer, num_layers); });
}

int specref_token_exit_test(const double* logits, int32_t v, int32_t drafted, int32_t k,
                            int32_t* out) {
  return guard([&] { *out = token_exit_test({logits, static_cast<size_t>(v)}, drafted, k); });
}

int specref_make_gate_plan(const faser_exit_policy* policy, const faser_gate_entry* batch,
                           int32_t n, double b, double r, int32_t num_layers,
                           faser_gate_plan* out) {
  return guard([&] {
    std::vector<GateEntry> entries(n);
    for (int i = 0; i < n; ++i) entries[i] = {batch[i].spec_length, batch[i].accept_estimate};
    auto g = make_gate_plan(to_policy(policy), entries, b, r, LatencyModel::default_ground_truth(),
                            num_layers);
    out->first_layer = g.first_layer;
    out->stop_layer = g.stop_layer;
    out->s_eff = g.s_eff;
  });
}

int specref_plan_overlap(int32_t s, int32_t b, const double* r_grid, int32_t n_r,
                         faser_overlap_plan* out) {
  return guard([&] {
    auto pl = plan_overlap(s, b, LatencyModel::default_ground_truth(),
                           {r_grid, static_cast<size_t>(n_r)});
    out->enabled = pl.enabled;
    out->chunk = pl.chunk;
    out->r = pl.r;
    out->predicted_ms = pl.predicted_ms;
    out->serial_ms = pl.serial_ms;
  });
}

int specref_eval_latency(int32_t stage, double b, double s, double r, double* out) {
  return guard([&] {
    auto m = LatencyModel::default_ground_truth();
    const PiecewiseLatencyParams* ps[4] = {&m.draft, &m.target, &m.ee_check, &m.prune};
    *out = eval_latency(*ps[stage], b, s, r);
  });
}

// ---- wire formats (workload.cpp:34-71, metrics.cpp:68-113): reference writers / parser, for the
// product's byte-for-byte format tests
int specref_write_trace(const char* path, int32_t n, const double* arrival_ms, const int32_t* in_len,
                        const int32_t* out_len) {
  return guard([&] {
    std::vector<TraceRecord> recs(n);
    for (int i = 0; i < n; ++i) recs[i] = {arrival_ms[i], in_len[i], out_len[i]};
    write_trace(path, recs);
  });
}
int specref_ingest_trace(const char* path, int32_t cap, double* arrival_ms, int32_t* in_len, int32_t* out_len,
                         int32_t* n) {
  return guard([&] {
    auto recs = ingest_trace(path);
    *n = static_cast<int32_t>(recs.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      arrival_ms[i] = recs[i].arrival_ms;
      in_len[i] = recs[i].input_len;
      out_len[i] = recs[i].output_len;
    }
  });
}
#ifdef SPECREF_METRICS
// Summary (metrics.hpp:34-66): ints = {requests, finished, total_output_tokens, drafted,
// submitted, accepted, wasted_draft_tokens, false_prunes, iterations, overlap_iterations},
// dbls = {makespan, throughput, mean_lat, p50_lat, p99_lat, mean_tpot, global_tpot, draft_ms,
// verify_ms, overhead_ms, verify_share, acceptance_ratio, layer_work, layer_work_full},
// hist = spec_length_hist pairs (n_hist x 2); writes metrics JSONL (summary only) + CSV.
int specref_write_summary(const char* jsonl_path, const char* csv_path, const char* mode, uint64_t seed,
                          const int64_t* ints, const double* dbls, const int64_t* hist, int32_t n_hist,
                          int32_t oracle_checked, int32_t oracle_ok) {
  return guard([&] {
    Metrics m;
    MetricsSummary& s = m.summary;
    s.mode = mode;
    s.seed = seed;
    s.requests = ints[0];
    s.finished = ints[1];
    s.total_output_tokens = ints[2];
    s.drafted_tokens = ints[3];
    s.submitted_tokens = ints[4];
    s.accepted_tokens = ints[5];
    s.wasted_draft_tokens = ints[6];
    s.false_prunes = ints[7];
    s.iterations = ints[8];
    s.overlap_iterations = ints[9];
    s.makespan_ms = dbls[0];
    s.throughput_tok_s = dbls[1];
    s.mean_request_latency_ms = dbls[2];
    s.p50_request_latency_ms = dbls[3];
    s.p99_request_latency_ms = dbls[4];
    s.mean_tpot_ms = dbls[5];
    s.global_tpot_ms = dbls[6];
    s.draft_time_ms = dbls[7];
    s.verify_time_ms = dbls[8];
    s.overhead_time_ms = dbls[9];
    s.verify_share = dbls[10];
    s.acceptance_ratio = dbls[11];
    s.layer_work = dbls[12];
    s.layer_work_full = dbls[13];
    for (int i = 0; i < n_hist; ++i) s.spec_length_hist.push_back({static_cast<int>(hist[2 * i]), hist[2 * i + 1]});
    s.oracle_checked = oracle_checked != 0;
    s.oracle_ok = oracle_ok != 0;
    write_metrics_jsonl(m, jsonl_path);
    write_summary_csv(s, csv_path);
  });
}

#endif  // SPECREF_METRICS

int specref_synth_prompt(uint64_t seed, int32_t index, int32_t len, int32_t vocab, int32_t* out) {
  return guard([&] {
    auto v = synth_prompt(seed, index, len, vocab);
    std::copy(v.begin(), v.end(), out);
  });
}

// Poisson arrivals over rate segments (workload.cpp:73-98). Returns count; arrays sized cap.
int specref_synth_workload(const double* seg_duration_ms, const double* seg_rate, int32_t n_seg,
                           int32_t in_lo, int32_t in_hi, int32_t out_lo, int32_t out_hi,
                           uint64_t seed, double* arrival_ms, int32_t* in_len, int32_t* out_len,
                           int32_t cap, int32_t* n_out) {
  return guard([&] {
    std::vector<RateSegment> segs(n_seg);
    for (int i = 0; i < n_seg; ++i) segs[i] = {seg_duration_ms[i], seg_rate[i]};
    auto recs = synth_workload(segs, {in_lo, in_hi}, {out_lo, out_hi}, seed);
    *n_out = static_cast<int32_t>(recs.size());
    for (int i = 0; i < static_cast<int>(recs.size()) && i < cap; ++i) {
      arrival_ms[i] = recs[i].arrival_ms;
      in_len[i] = recs[i].input_len;
      out_len[i] = recs[i].output_len;
    }
  });
}

int specref_sine_segments(double mean_rate, double ptv, double duration_ms, int32_t steps,
                          double* seg_duration_ms, double* seg_rate) {
  return guard([&] {
    auto s = sine_segments(mean_rate, ptv, duration_ms, steps);
    for (int i = 0; i < steps; ++i) {
      seg_duration_ms[i] = s[i].duration_ms;
      seg_rate[i] = s[i].rate_per_s;
    }
  });
}

// ------------------------------------------------------------------ episode runner

// Per-request speculative length schedule used for bit-exact dynamic-k runs (config 2):
// k = S[h % |S|], h = hash_combine(hash_combine(mix64(seed), req_id + 1), round + 1),
// S = DrafterConfig::candidates (drafter.hpp:16). bench.py / tests restate it in Python.
/* The reference's own AcceptanceWindow (sdcore.cpp:8-35): pushes n rounds (s, submitted,
 * accepted) with the given window and, after each push, evaluates rate_for(q) for the nq query
 * lengths and overall(): out[i * (nq + 1) + j] (j = nq is overall). */
int specref_acceptance_window_replay(const int32_t* s, const int32_t* submitted, const int32_t* accepted,
                                     int32_t n, int32_t window, const int32_t* qs, int32_t nq, double* out) {
  specsim::AcceptanceWindow w;
  for (int i = 0; i < n; ++i) {
    w.push({s[i], submitted[i], accepted[i]}, window);
    for (int j = 0; j < nq; ++j) out[static_cast<size_t>(i) * (nq + 1) + j] = w.rate_for(qs[j]);
    out[static_cast<size_t>(i) * (nq + 1) + nq] = w.overall();
  }
  return 0;
}

// ------------------------------------------------------------------ AdaptiveDrafter
// The reference's own AdaptiveDrafter / GpPosterior / AcceptanceBook (drafter.cpp, compiled in
// place against oracle/eigen_shim for its three Eigen calls) behind the same glue the product's
// faser_drafter_* applies for the missing sim loop (include/faser/engine.h): per round each
// request's (spec, submitted, accepted) is pushed into its AcceptanceWindow (W = window_request),
// rounds with submitted > 0 record their ratio in the AcceptanceBook under the round number
// rounds_in(key) + 1, and observe_round gets the mean ratio per distinct spec length.
namespace {
specsim::PiecewiseLatencyParams to_params(const faser_latency_params& p) {
  specsim::PiecewiseLatencyParams q;
  q.stage = static_cast<specsim::StageKind>(p.stage);
  q.knee = p.knee;
  q.a1 = p.a1;
  q.gamma1 = p.gamma1;
  q.a2 = p.a2;
  q.gamma2 = p.gamma2;
  q.c0 = p.c0;
  q.c1 = p.c1;
  q.c2 = p.c2;
  return q;
}
struct RefDrafter {
  specsim::LatencyModel models;
  specsim::DrafterConfig cfg;
  specsim::AcceptanceBook book;
  specsim::AdaptiveDrafter drafter;
  std::map<int64_t, specsim::Request> reqs;
  RefDrafter(const specsim::DrafterConfig& c, const specsim::LatencyModel& m)
      : models(m), cfg(c), book(c.window_ctx, c.cold_start_accept), drafter(c, &models) {}
};
}  // namespace

void* specref_drafter_create(const faser_drafter_cfg* c, const faser_latency_model* m) {
  specsim::DrafterConfig cfg;
  cfg.candidates.assign(c->candidates, c->candidates + c->n_candidates);
  cfg.epsilon = c->epsilon;
  cfg.window_ctx = c->window_ctx;
  cfg.window_request = c->window_request;
  cfg.kernel_len = c->kernel_len;
  cfg.kernel_var = c->kernel_var;
  cfg.noise_var = c->noise_var;
  cfg.cold_start_accept = c->cold_start_accept;
  specsim::LatencyModel lm = specsim::LatencyModel::default_ground_truth();
  if (m) {
    lm.draft = to_params(m->draft);
    lm.target = to_params(m->target);
    lm.ee_check = to_params(m->ee_check);
    lm.prune = to_params(m->prune);
  }
  return new RefDrafter(cfg, lm);
}
void specref_drafter_destroy(void* h) { delete static_cast<RefDrafter*>(h); }

int specref_drafter_assign(void* h, const int64_t* ids, int32_t n, int32_t b, double r, int32_t* out) {
  auto* d = static_cast<RefDrafter*>(h);
  std::vector<const specsim::Request*> batch;
  for (int i = 0; i < n; ++i) {
    specsim::Request& q = d->reqs[ids[i]];
    q.id = static_cast<int>(ids[i]);
    batch.push_back(&q);
  }
  try {
    const std::vector<int> k = d->drafter.assign_lengths(batch, b, r, d->book);
    for (int i = 0; i < n; ++i) out[i] = k[i];
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

int specref_drafter_observe(void* h, int32_t b, double r, double t_obs_ms, const int64_t* ids, const int32_t* spec,
                            const int32_t* submitted, const int32_t* accepted, int32_t n) {
  auto* d = static_cast<RefDrafter*>(h);
  const specsim::ContextKey key = specsim::ContextKey::of(b, r);
  const int round = d->drafter.rounds_in(key) + 1;
  std::map<int, std::pair<double, int>> by_s;
  for (int i = 0; i < n; ++i) {
    specsim::Request& q = d->reqs[ids[i]];
    q.accept_window.push({spec[i], submitted[i], accepted[i]}, d->cfg.window_request);
    if (submitted[i] > 0) {
      const double ratio = static_cast<double>(accepted[i]) / submitted[i];
      d->book.record(key, round, spec[i], ratio);
      auto& e = by_s[spec[i]];
      e.first += ratio;
      e.second += 1;
    }
  }
  std::vector<std::pair<int, double>> acc;
  for (const auto& [s, e] : by_s) acc.emplace_back(s, e.first / e.second);
  try {
    d->drafter.observe_round(b, r, t_obs_ms, acc);
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

int specref_drafter_posterior(void* h, int32_t b, double r, double* mu, double* sigma, int32_t* rounds) {
  auto* d = static_cast<RefDrafter*>(h);
  const specsim::ContextKey key = specsim::ContextKey::of(b, r);
  const specsim::GpPosterior* gp = d->drafter.find_posterior(key);
  for (size_t i = 0; i < d->cfg.candidates.size(); ++i) {
    const int s = d->cfg.candidates[i];
    mu[i] = gp ? gp->mu(s, d->cfg) : 0.0;
    sigma[i] = gp ? gp->sigma(s, d->cfg) : std::sqrt(d->cfg.kernel_var);
  }
  *rounds = d->drafter.rounds_in(key);
  return 0;
}

int32_t specref_sched_k(uint64_t seed, int64_t req_id, int32_t round) {
  static const int kS[8] = {1, 2, 3, 4, 5, 6, 8, 10};
  const uint64_t h = hash_combine(hash_combine(mix64(seed), static_cast<uint64_t>(req_id) + 1),
                                  static_cast<uint64_t>(round) + 1);
  return kS[h % 8];
}



// Runs the serving loop over a backlog: iteration-boundary admission in index order
// (B_max cap), per live request draft_tokens -> verify -> commit
// (SPEC.md:545-549), exempt-position rule, finished requests leave after the round.
// out_tokens: [n_requests][out_cap]; round_log (nullable): records in (round, batch order).
int specref_run_episode(const specref_episode_cfg* cfg, const int32_t* prompt_tokens,
                        const int64_t* prompt_off, const int32_t* max_out, int32_t* out_tokens,
                        int32_t out_cap, int32_t* out_len, faser_round_result* round_log,
                        int64_t log_cap, int64_t* n_log, specref_episode_stats* stats) {
  return guard([&] {
    LayeredToyLM model(to_params(&cfg->model));
    SpeculativeEngine eng(&model);
    const ExitPolicy policy = to_policy(&cfg->policy);
    GatePlan gate;
    gate.first_layer = cfg->gate.first_layer;
    gate.stop_layer = cfg->gate.stop_layer;
    gate.s_eff = cfg->gate.s_eff;

    const int n = cfg->n_requests;
    std::vector<Request> reqs(n);
    for (int i = 0; i < n; ++i) {
      auto r = row(prompt_tokens, prompt_off, i);
      reqs[i].id = i;
      reqs[i].prompt.assign(r.begin(), r.end());
      reqs[i].max_out = max_out[i];
      reqs[i].done = max_out[i] <= 0;
    }
    std::vector<int> req_round(n, 0);
    std::vector<double> t_first(n, -1.0), t_last(n, -1.0);
    std::vector<faser_round_result> results;  // per batch position, this round

    std::vector<int> live;
    int next = 0;
    int64_t logged = 0;
    specref_episode_stats st{};
    const int T = std::max(1, cfg->threads);

    auto work_one = [&](int pos) {
      const int id = live[pos];
      Request& req = reqs[id];
      const int k = cfg->k_mode == 1 ? specref_sched_k(cfg->k_seed, id, req_round[id]) : cfg->fixed_k;
      faser_round_result& rr = results[pos];
      std::memset(&rr, 0, sizeof(rr));
      rr.req_id = id;
      rr.spec_length = k;
      auto drafted = eng.draft_tokens(req, k);
      rr.drafted = static_cast<int32_t>(drafted.size());
      VerifyOutcome o = cfg->early_exit ? eng.verify_with_early_exit(req, drafted, policy, gate)
                                        : eng.full_verify(req, drafted);
      to_c(o, &rr.outcome);
      const int before = static_cast<int>(req.committed.size());
      rr.committed = eng.commit(req, o, drafted);
      for (int j = 0; j < rr.committed; ++j) rr.tokens[j] = req.committed[before + j];
      if (cfg->exempt_rule) req.exempt_position = o.pruned_at ? before + o.pruned_at->first : -1;
      rr.done = req.done;
      rr.exempt_position = req.exempt_position;
      rr.n_committed_total = static_cast<int32_t>(req.committed.size());
      req_round[id] += 1;
    };

    // Persistent pool: worker w handles batch positions w, w+T, ...; two barrier phases
    // per round (start, end). The main thread is worker 0.
    std::atomic<bool> stop{false};
    SpinBarrier sync(T);
    auto worker = [&](int w) {
      for (;;) {
        sync.arrive_and_wait();  // round start
        if (stop.load(std::memory_order_acquire)) return;
        for (int pos = w; pos < static_cast<int>(live.size()); pos += T) work_one(pos);
        sync.arrive_and_wait();  // round end
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < T; ++w) pool.emplace_back(worker, w);

    const auto t0 = std::chrono::steady_clock::now();
    int64_t round = 0;
    std::exception_ptr err;
    try {
      for (;;) {
        while (next < n && static_cast<int>(live.size()) < cfg->max_batch) {
          if (!reqs[next].done) live.push_back(next);
          ++next;
        }
        if (live.empty()) break;
        if (cfg->max_rounds > 0 && round >= cfg->max_rounds) break;
        results.assign(live.size(), faser_round_result{});
        sync.arrive_and_wait();
        for (int pos = 0; pos < static_cast<int>(live.size()); pos += T) work_one(pos);
        sync.arrive_and_wait();
        const double now_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::vector<int> keep;
        for (size_t pos = 0; pos < live.size(); ++pos) {
          const auto& rr = results[pos];
          const int id = live[pos];
          st.drafted += rr.drafted;
          st.submitted += rr.outcome.submitted;
          st.accepted += rr.outcome.accepted_count;
          st.committed += rr.committed;
          st.false_prunes += rr.outcome.false_prune;
          st.layer_work += rr.outcome.full_layers_run;
          st.layer_work_full += static_cast<double>(cfg->model.layers) * rr.outcome.submitted;
          if (rr.committed > 0) {
            if (t_first[id] < 0) t_first[id] = now_ms;
            t_last[id] = now_ms;
          }
          if (round_log && logged < log_cap) round_log[logged] = rr;
          ++logged;
          if (!rr.done) keep.push_back(id);
        }
        live.swap(keep);
        ++round;
      }
    } catch (...) {
      err = std::current_exception();
    }
    stop.store(true, std::memory_order_release);
    sync.arrive_and_wait();
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);

    st.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    st.rounds = round;
    std::vector<double> tpots;
    double mean = 0.0;
    for (int i = 0; i < n; ++i) {
      const auto& c = reqs[i].committed;
      out_len[i] = static_cast<int32_t>(c.size());
      for (int j = 0; j < static_cast<int>(c.size()) && j < out_cap; ++j)
        out_tokens[static_cast<int64_t>(i) * out_cap + j] = c[j];
      if (reqs[i].done) ++st.finished;
      if (c.size() >= 2 && t_first[i] >= 0) {
        tpots.push_back((t_last[i] - t_first[i]) / static_cast<double>(c.size() - 1));
      }
    }
    if (!tpots.empty()) {
      std::sort(tpots.begin(), tpots.end());
      st.p50_tpot_ms = tpots[tpots.size() / 2];
      for (double t : tpots) mean += t;
      st.mean_tpot_ms = mean / tpots.size();
    }
    if (n_log) *n_log = logged;
    if (stats) *stats = st;
  });
}

}  // extern "C"

// controllers.cpp — host-side scalar controllers of the data path (no device work).
//
// Native restatements of the reference's per-batch scalar math that feeds the GPU step:
//   ExitPolicy::k_at          exitctl.cpp:9-17
//   estimate_prunable, effective_saving(_from), should_prune, make_gate_plan
//                             exitctl.cpp:19-82
//   eval_latency + default_ground_truth
//                             latmodel.cpp:32-62, 396-403
//   predict_pipeline_ms, plan_overlap
//                             overlap.cpp:9-42
//   synth_prompt              workload.cpp:116-122 (+ rng.hpp:41-79)
//   synth_workload, sine_segments
//                             workload.cpp:73-114 (+ SplitMixStream::next_exp, rng.hpp:55-59)
// All double arithmetic is written in the reference's evaluation order; this TU is built
// without FMA contraction (-ffp-contract=off) so results are bit-identical to the x86-64
// reference build (tests/test_controllers.py checks against oracle/_ref).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>

#include "faser/engine.h"

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;
uint64_t mix64(uint64_t x) {
  x += kGamma;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t substream(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }

bool valid_policy(const faser_exit_policy* p) {
  return p && p->k_init >= 1 && p->k_final >= 1 && p->k_final <= p->k_init;
}

int k_at(const faser_exit_policy& p, int layer, int num_layers) {
  if (layer <= p.l_init || num_layers <= p.l_init) return p.k_init;
  if (layer >= num_layers) return p.k_final;
  const double t = static_cast<double>(layer - p.l_init) / static_cast<double>(num_layers - p.l_init);
  const int k = static_cast<int>(std::lround(p.k_init + (p.k_final - p.k_init) * t));
  return std::max(1, k);
}

// own_share (latmodel.cpp:32-42): draft/prune run on r, target/ee_check on 1-r.
double own_share(int stage, double r) { return (stage == 0 || stage == 3) ? r : 1.0 - r; }

// eval_latency = piecewise_factor(own share) * load_term (latmodel.cpp:44-62).
bool eval(const faser_latency_params& p, double b, double s, double r, double* out) {
  const double x = own_share(p.stage, r);
  if (!(x > 0.0) || x > 1.0) return false;  // std::invalid_argument in the reference
  const double factor = x <= p.knee ? p.a1 - p.gamma1 * x : p.a2 - p.gamma2 * x;
  double load;
  switch (p.stage) {
    case 0: load = p.c0 * b + p.c1 * s + p.c2; break;
    case 1: load = (p.c0 * b + p.c1) * s + p.c2; break;
    default: load = p.c0 * b * s + p.c1; break;
  }
  *out = factor * load;
  return true;
}

faser_latency_model default_model() {
  faser_latency_model m{};
  m.draft = {0, 0, 0.5, 1.6, 0.9, 1.275, 0.25, 0.003, 0.28, 0.5};
  m.target = {1, 0, 0.5, 1.5, 0.8, 1.2, 0.2, 0.008, 0.18, 0.3};
  m.ee_check = {2, 0, 0.5, 1.6, 1.0, 1.3, 0.4, 2e-6, 0.002, 0.0};
  m.prune = {3, 0, 0.6, 1.5, 1.0, 1.2, 0.5, 2e-6, 0.003, 0.0};
  return m;
}

}  // namespace

extern "C" {

int32_t faser_abi_version(void) { return FASER_ABI_VERSION; }

faser_status faser_abi_struct_sizes(int64_t* out, int32_t n) {
  if (!out) return FASER_EINVAL;
  const int64_t sizes[15] = {
      sizeof(faser_toy_params),    sizeof(faser_exit_policy),   sizeof(faser_gate_plan),
      sizeof(faser_gate_entry),    sizeof(faser_overlap_plan),  sizeof(faser_latency_params),
      sizeof(faser_latency_model), sizeof(faser_verify_outcome), sizeof(faser_model_desc),
      sizeof(faser_engine_cfg),    sizeof(faser_step_plan),     sizeof(faser_round_result),
      sizeof(faser_llama_shape),   sizeof(faser_timeline_event), sizeof(faser_timeline_info)};
  for (int i = 0; i < n && i < 15; ++i) out[i] = sizes[i];
  return FASER_OK;
}

faser_status faser_k_table(const faser_exit_policy* policy, int32_t num_layers, int32_t* table) {
  if (!valid_policy(policy) || !table || num_layers < 1 || num_layers > FASER_MAX_LAYERS)
    return FASER_EINVAL;
  for (int l = 0; l <= num_layers; ++l) table[l] = k_at(*policy, l, num_layers);
  return FASER_OK;
}

void faser_default_latency_model(faser_latency_model* out) {
  if (out) *out = default_model();
}

faser_status faser_eval_latency(const faser_latency_model* m, int32_t stage, double b, double s,
                                double r, double* out_ms) {
  if (!out_ms || stage < 0 || stage > 3) return FASER_EINVAL;
  const faser_latency_model mm = m ? *m : default_model();
  const faser_latency_params* ps[4] = {&mm.draft, &mm.target, &mm.ee_check, &mm.prune};
  return eval(*ps[stage], b, s, r, out_ms) ? FASER_OK : FASER_EINVAL;
}

// make_gate_plan (exitctl.cpp:70-82) with should_prune (:48-54), effective_saving (:29-46)
// and estimate_prunable (:19-27) inlined in reference order.
faser_status faser_make_gate_plan(const faser_exit_policy* policy, const faser_gate_entry* batch,
                                  int32_t n, double b, double r, const faser_latency_model* models,
                                  int32_t num_layers, faser_gate_plan* out) {
  if (!policy || !out || (n > 0 && !batch)) return FASER_EINVAL;
  const faser_latency_model m = models ? *models : default_model();
  double prunable = 0.0;
  for (int i = 0; i < n; ++i) {
    const double a = batch[i].accept_estimate;
    if (a < 0.0 || a > 1.0) return FASER_EINVAL;
    prunable += batch[i].spec_length * (1.0 - a);
  }
  const double s_eff = std::max(prunable, 1.0);
  out->first_layer = policy->l_init;
  out->stop_layer = policy->l_init;
  out->s_eff = s_eff;
  if (policy->l_init > num_layers || policy->l_init < 1 || n == 0) return FASER_OK;
  int layer = policy->l_init;
  while (layer < num_layers) {
    if (layer < 1 || layer > num_layers) return FASER_EINVAL;
    double t_ee, t_target, t_prune;
    if (!eval(m.ee_check, b, s_eff, r, &t_ee) || !eval(m.target, b, s_eff, r, &t_target) ||
        !eval(m.prune, b, s_eff, r, &t_prune))
      return FASER_EINVAL;
    if (!(t_target > 0.0)) return FASER_EINVAL;
    const double est_layers = num_layers * t_ee / t_target;
    const double remaining = std::max(static_cast<double>(num_layers - layer) - est_layers, 0.0);
    const double save_ms = remaining / num_layers * t_target;
    if (!(save_ms > t_prune)) break;
    ++layer;
  }
  out->stop_layer = layer;
  return FASER_OK;
}

// plan_overlap (overlap.cpp:23-42) with predict_pipeline_ms (:9-21).
faser_status faser_plan_overlap(int32_t s, int32_t b, const faser_latency_model* models,
                                const double* r_grid, int32_t n_r, faser_overlap_plan* out) {
  if (!out || s < 1 || (n_r > 0 && !r_grid)) return FASER_EINVAL;
  const faser_latency_model m = models ? *models : default_model();
  double d1, t0;
  if (!eval(m.draft, b, s, 1.0, &d1) || !eval(m.target, b, s, 0.0, &t0)) return FASER_EINVAL;
  out->enabled = 0;
  out->chunk = 0;
  out->r = 1.0;
  out->serial_ms = d1 + t0;
  out->predicted_ms = out->serial_ms;
  double best = std::numeric_limits<double>::infinity();
  for (int chunk = 1; chunk <= s; ++chunk) {
    for (int i = 0; i < n_r; ++i) {
      const double r = r_grid[i];
      double draft_t = 0.0, verify_t = 0.0;
      int remaining = s;
      while (remaining > 0) {
        const int c = std::min(chunk, remaining);
        remaining -= c;
        double dm, tm;
        if (!eval(m.draft, b, c, r, &dm) || !eval(m.target, b, c, r, &tm)) return FASER_EINVAL;
        draft_t += dm;
        verify_t = std::max(verify_t, draft_t) + tm;
      }
      if (verify_t < out->serial_ms && verify_t < best) {
        best = verify_t;
        out->enabled = 1;
        out->chunk = chunk;
        out->r = r;
        out->predicted_ms = verify_t;
      }
    }
  }
  return FASER_OK;
}

faser_status faser_synth_prompt(uint64_t seed, int32_t index, int32_t len, int32_t vocab,
                                int32_t* out) {
  if (!out || vocab < 2) return FASER_EINVAL;
  const int n = std::max(len, 1);
  uint64_t state = mix64(substream(substream(seed, 0x70726d70ull), static_cast<uint64_t>(index)));
  const uint64_t span = static_cast<uint64_t>(vocab - 2) + 1;
  for (int i = 0; i < n; ++i) {
    state += kGamma;
    out[i] = static_cast<int32_t>(mix64(state) % span);
  }
  return FASER_OK;
}

faser_status faser_synth_workload(const double* seg_duration_ms, const double* seg_rate_per_s,
                                  int32_t n_seg, int32_t in_lo, int32_t in_hi, int32_t out_lo,
                                  int32_t out_hi, uint64_t seed, double* arrival_ms,
                                  int32_t* in_len, int32_t* out_len, int32_t cap, int32_t* n) {
  if (!n || n_seg < 0 || (n_seg > 0 && (!seg_duration_ms || !seg_rate_per_s)) || cap < 0 ||
      (cap > 0 && (!arrival_ms || !in_len || !out_len)) || in_hi < in_lo || out_hi < out_lo)
    return FASER_EINVAL;
  // two counter streams (SplitMixStream: state = mix64(seed); draw = mix64(state += gamma))
  uint64_t arrv = mix64(substream(seed, 0x61727276ull));  // "arrv"
  uint64_t lens = mix64(substream(seed, 0x6c656e73ull));  // "lens"
  auto next_u64 = [](uint64_t& st) {
    st += kGamma;
    return mix64(st);
  };
  auto next_exp = [&](double rate) {
    double u = static_cast<double>(next_u64(arrv) >> 11) * 0x1.0p-53;
    if (u <= 0.0) u = 0x1.0p-53;
    return -std::log(u) / rate;
  };
  auto next_int = [&](int lo, int hi) {
    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
    return lo + static_cast<int>(next_u64(lens) % span);
  };
  int32_t count = 0;
  double seg_start = 0.0;
  for (int i = 0; i < n_seg; ++i) {
    if (seg_duration_ms[i] < 0) return FASER_EINVAL;  // std::invalid_argument in the reference
    const double seg_end = seg_start + seg_duration_ms[i];
    if (seg_rate_per_s[i] > 0.0) {
      const double rate_per_ms = seg_rate_per_s[i] / 1000.0;
      double t = seg_start + next_exp(rate_per_ms);
      while (t < seg_end) {
        const int a = next_int(in_lo, in_hi);
        const int b = next_int(out_lo, out_hi);
        if (count < cap) {
          arrival_ms[count] = t;
          in_len[count] = a;
          out_len[count] = b;
        }
        ++count;
        t += next_exp(rate_per_ms);
      }
    }
    seg_start = seg_end;
  }
  *n = count;
  return FASER_OK;
}

faser_status faser_sine_segments(double mean_rate_per_s, double peak_to_valley, double duration_ms,
                                 int32_t steps, double* seg_duration_ms, double* seg_rate_per_s) {
  if (steps < 1 || !(mean_rate_per_s > 0) || !(peak_to_valley >= 1) || !seg_duration_ms || !seg_rate_per_s)
    return FASER_EINVAL;
  const double a = (peak_to_valley - 1.0) / (peak_to_valley + 1.0);
  for (int i = 0; i < steps; ++i) {
    const double phase = 2.0 * 3.14159265358979323846 * (i + 0.5) / steps;
    seg_duration_ms[i] = duration_ms / steps;
    seg_rate_per_s[i] = mean_rate_per_s * (1.0 + a * std::sin(phase));
  }
  return FASER_OK;
}

}  // extern "C"

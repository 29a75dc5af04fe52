// drafter.cpp — the per-request speculative-length controller (host C++, no device work).
//
// Restates the reference's AdaptiveDrafter (drafter.hpp:98-129, drafter.cpp:175-220), its
// GpPosterior (drafter.cpp:34-97), AcceptanceBook (drafter.cpp:123-161) and the per-request
// AcceptanceWindow (sdcore.cpp:8-35) natively. The reference solves the GP with an Eigen LLT
// over the raw observation window (up to window_ctx x |S| points); observations only ever sit
// on the |S| candidate indices, so the same posterior follows exactly from per-candidate
// sufficient statistics (counts D, centred sums s):
//   mu(c)  = ybar + k_c^T (D K + s_n^2 I)^-1 s
//   var(c) = k_var - k_c^T (D K + s_n^2 I)^-1 D k_c
// (push-through identity on K_nn = A K A^T), an |S| x |S| solve instead of an n x n LLT.
// Parity: the reference TU cannot be compiled here (Eigen absent) -> unpinned; the tests check
// this against a numpy restatement of the raw-window LLT (tests/test_drafter.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "faser/engine.h"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxS = 16;

struct Key {
  int batch_log2 = 0, sm_decile = 10;
  bool operator<(const Key& o) const {
    return std::tie(batch_log2, sm_decile) < std::tie(o.batch_log2, o.sm_decile);
  }
};

// ContextKey::of (drafter.cpp:25-32)
Key key_of(int batch, double r) {
  Key k;
  k.batch_log2 = static_cast<int>(std::lround(std::log2(static_cast<double>(batch))));
  k.sm_decile = std::clamp(static_cast<int>(std::lround(r * 10.0)), 1, 10);
  return k;
}

double beta_of(int n_cand, int round) {  // drafter.cpp:14-17
  const int n = std::max(round, 1);
  return 2.0 * std::log(n_cand * static_cast<double>(n) * n * kPi * kPi / 6.0);
}

// Solves M x = b for a small dense system (partial pivoting). M is m x m row-major.
void solve(std::vector<double> M, std::vector<double> b, int m, std::vector<double>* x) {
  for (int c = 0; c < m; ++c) {
    int p = c;
    for (int r = c + 1; r < m; ++r)
      if (std::fabs(M[r * m + c]) > std::fabs(M[p * m + c])) p = r;
    if (p != c) {
      for (int j = 0; j < m; ++j) std::swap(M[c * m + j], M[p * m + j]);
      std::swap(b[c], b[p]);
    }
    for (int r = c + 1; r < m; ++r) {
      const double f = M[r * m + c] / M[c * m + c];
      if (f == 0.0) continue;
      for (int j = c; j < m; ++j) M[r * m + j] -= f * M[c * m + j];
      b[r] -= f * b[c];
    }
  }
  x->assign(m, 0.0);
  for (int r = m - 1; r >= 0; --r) {
    double a = b[r];
    for (int j = r + 1; j < m; ++j) a -= M[r * m + j] * (*x)[j];
    (*x)[r] = a / M[r * m + r];
  }
}

struct Gp {
  struct Obs {
    int index;
    double cost;
    int round;
  };
  std::vector<Obs> window;
  std::vector<double> mu, sigma;
  bool dirty = true;

  void observe(int index, double cost, int round, int window_ctx) {  // drafter.cpp:34-44
    window.push_back({index, cost, round});
    window.erase(std::remove_if(window.begin(), window.end(),
                                [&](const Obs& o) { return o.round <= round - window_ctx; }),
                 window.end());
    dirty = true;
  }

  void recompute(const faser_drafter_cfg& cfg) {  // drafter.cpp:46-80
    const int m = cfg.n_candidates;
    mu.assign(m, 0.0);
    sigma.assign(m, std::sqrt(cfg.kernel_var));
    dirty = false;
    const int n = static_cast<int>(window.size());
    if (n == 0) return;
    double mean = 0.0;
    for (const Obs& o : window) mean += o.cost;
    mean /= n;
    std::vector<double> cnt(m, 0.0), sum(m, 0.0);
    for (const Obs& o : window) {
      cnt[o.index] += 1.0;
      sum[o.index] += o.cost - mean;
    }
    const double ls2 = 2.0 * cfg.kernel_len * cfg.kernel_len;
    auto kern = [&](int a, int b) {
      const double d = a - b;
      return cfg.kernel_var * std::exp(-d * d / ls2);
    };
    std::vector<double> A(m * m);  // D K + s_n^2 I
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) A[i * m + j] = cnt[i] * kern(i, j) + (i == j ? cfg.noise_var : 0.0);
    std::vector<double> alpha;
    solve(A, sum, m, &alpha);
    for (int c = 0; c < m; ++c) {
      double kd = 0.0;
      std::vector<double> dk(m);
      for (int i = 0; i < m; ++i) {
        kd += kern(c, i) * alpha[i];
        dk[i] = cnt[i] * kern(c, i);
      }
      mu[c] = mean + kd;
      std::vector<double> y;
      solve(A, dk, m, &y);
      double q = 0.0;
      for (int i = 0; i < m; ++i) q += kern(c, i) * y[i];
      sigma[c] = std::sqrt(std::max(cfg.kernel_var - q, 1e-12));
    }
  }
};

struct ReqWindow {  // AcceptanceWindow (sdcore.cpp:8-35)
  struct E {
    int s, submitted, accepted;
  };
  std::deque<E> entries;
  double rate_for(int s) const {
    double acc = 0.0;
    int n = 0;
    for (const E& e : entries)
      if (e.s == s && e.submitted > 0) {
        acc += static_cast<double>(e.accepted) / e.submitted;
        ++n;
      }
    return n ? acc / n : -1.0;
  }
  double overall() const {
    double acc = 0.0;
    int n = 0;
    for (const E& e : entries)
      if (e.submitted > 0) {
        acc += static_cast<double>(e.accepted) / e.submitted;
        ++n;
      }
    return n ? acc / n : -1.0;
  }
};

struct Ctx {
  Gp gp;
  int rounds = 0;
  std::map<int, std::deque<std::pair<int, double>>> latency;  // s -> (round, ms)
  std::deque<std::tuple<int, int, double>> book;              // AcceptanceBook window
};

}  // namespace

struct faser_drafter {
  faser_drafter_cfg cfg{};
  faser_latency_model models{};
  std::map<Key, Ctx> ctx;
  std::unordered_map<int64_t, ReqWindow> req;

  int index_of(int s) const {
    for (int i = 0; i < cfg.n_candidates; ++i)
      if (cfg.candidates[i] == s) return i;
    return -1;
  }
  double context_rate(const Ctx& c, int s) const {
    double acc = 0.0;
    int n = 0;
    for (const auto& [round, ss, ratio] : c.book)
      if (ss == s) {
        acc += ratio;
        ++n;
      }
    return n ? acc / n : -1.0;
  }
  double context_overall(const Ctx& c) const {
    if (c.book.empty()) return -1.0;
    double acc = 0.0;
    for (const auto& [round, ss, ratio] : c.book) acc += ratio;
    return acc / c.book.size();
  }
  // AcceptanceBook::estimate (drafter.cpp:151-161)
  double estimate(int64_t id, const Ctx& c, int s) const {
    auto it = req.find(id);
    double v = it != req.end() ? it->second.rate_for(s) : -1.0;
    if (v >= 0.0) return v;
    v = context_rate(c, s);
    if (v >= 0.0) return v;
    v = context_overall(c);
    if (v >= 0.0) return v;
    v = it != req.end() ? it->second.overall() : -1.0;
    if (v >= 0.0) return v;
    return cfg.cold_start_accept;
  }
  // AdaptiveDrafter::latency_estimate (drafter.cpp:163-173): windowed mean, else the model's
  // serial_iteration_ms = draft(b, s, r=1) + target(b, s, r=0) (latmodel.hpp:104-106).
  double latency_estimate(const Ctx& c, int b, int s) const {
    auto it = c.latency.find(s);
    if (it != c.latency.end() && it->second.size() >= 3) {
      double acc = 0.0;
      for (const auto& [round, ms] : it->second) acc += ms;
      return acc / it->second.size();
    }
    double d = 0.0, t = 0.0;
    faser_eval_latency(&models, 0, b, s, 1.0, &d);
    faser_eval_latency(&models, 1, b, s, 0.0, &t);
    return d + t;
  }
};

extern "C" {

void faser_drafter_default_cfg(faser_drafter_cfg* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  const int s[8] = {1, 2, 3, 4, 5, 6, 8, 10};
  out->n_candidates = 8;
  for (int i = 0; i < 8; ++i) out->candidates[i] = s[i];
  out->window_ctx = 64;
  out->window_request = 16;
  out->epsilon = 1e-6;
  out->kernel_len = 1.0;
  out->kernel_var = 1.0;
  out->noise_var = 0.1;
  out->cold_start_accept = 0.7;
}

faser_status faser_drafter_create(const faser_drafter_cfg* cfg, const faser_latency_model* models,
                                  faser_drafter** out) {
  if (!out) return FASER_EINVAL;
  *out = nullptr;
  faser_drafter_cfg c;
  if (cfg) {
    c = *cfg;
  } else {
    faser_drafter_default_cfg(&c);
  }
  if (c.n_candidates < 1 || c.n_candidates > kMaxS || c.window_ctx < 1 || c.window_request < 1 ||
      !(c.kernel_len > 0) || !(c.kernel_var > 0) || !(c.noise_var > 0))
    return FASER_EINVAL;
  for (int i = 0; i < c.n_candidates; ++i)
    if (c.candidates[i] < 1 || c.candidates[i] > FASER_MAX_SPEC) return FASER_EINVAL;
  faser_drafter* d = new faser_drafter();
  d->cfg = c;
  if (models) {
    d->models = *models;
  } else {
    faser_default_latency_model(&d->models);
  }
  *out = d;
  return FASER_OK;
}

void faser_drafter_destroy(faser_drafter* d) { delete d; }

faser_status faser_drafter_set_models(faser_drafter* d, const faser_latency_model* models) {
  if (!d || !models) return FASER_EINVAL;
  d->models = *models;
  return FASER_OK;
}

double faser_drafter_beta(const faser_drafter_cfg* cfg, int32_t round) {
  return beta_of(cfg ? cfg->n_candidates : 8, round);
}

faser_status faser_drafter_objective(double t_hat_ms, int32_t s, double a_hat, double epsilon, double* out) {
  if (!out || !(t_hat_ms > 0.0) || s < 1) return FASER_EINVAL;  // std::invalid_argument
  *out = t_hat_ms / (s * a_hat + epsilon);
  return FASER_OK;
}

faser_status faser_drafter_assign(faser_drafter* d, const int64_t* req_ids, int32_t n, int32_t b, double r,
                                  int32_t* k_out) {
  if (!d || (n > 0 && (!req_ids || !k_out)) || b < 1) return FASER_EINVAL;
  const faser_drafter_cfg& cfg = d->cfg;
  Ctx& c = d->ctx[key_of(b, r)];
  const int m = cfg.n_candidates;
  if (c.rounds < m) {  // cold start: sweep the candidates round-robin (drafter.cpp:182-186)
    for (int i = 0; i < n; ++i) k_out[i] = cfg.candidates[c.rounds % m];
    return FASER_OK;
  }
  if (c.gp.dirty) c.gp.recompute(cfg);
  const double root_beta = std::sqrt(beta_of(m, c.rounds + 1));
  for (int i = 0; i < n; ++i) {
    int best = cfg.candidates[0];
    double best_lcb = std::numeric_limits<double>::infinity();
    for (int j = 0; j < m; ++j) {
      const int s = cfg.candidates[j];
      const double a_hat = d->estimate(req_ids[i], c, s);
      const double t_hat = d->latency_estimate(c, b, s);
      if (!(t_hat > 0.0)) return FASER_EINVAL;
      const double cost = t_hat / (s * a_hat + cfg.epsilon);
      const double lcb = cost - root_beta * c.gp.sigma[j];
      if (lcb < best_lcb) {  // strict '<': ties keep the smaller length
        best_lcb = lcb;
        best = s;
      }
    }
    k_out[i] = best;
  }
  return FASER_OK;
}

faser_status faser_drafter_observe(faser_drafter* d, int32_t b, double r, double t_obs_ms, const int64_t* req_ids,
                                   const int32_t* spec, const int32_t* submitted, const int32_t* accepted,
                                   int32_t n) {
  if (!d || b < 1 || !(t_obs_ms > 0.0) || (n > 0 && (!req_ids || !spec || !submitted || !accepted)))
    return FASER_EINVAL;
  const faser_drafter_cfg& cfg = d->cfg;
  Ctx& c = d->ctx[key_of(b, r)];
  const int round = c.rounds + 1;
  std::map<int, std::pair<double, int>> by_s;  // s -> (sum ratio, count)
  for (int i = 0; i < n; ++i) {
    if (d->index_of(spec[i]) < 0) return FASER_EINVAL;  // length not in the candidate set
    ReqWindow& w = d->req[req_ids[i]];
    w.entries.push_back({spec[i], submitted[i], accepted[i]});
    while (static_cast<int>(w.entries.size()) > cfg.window_request) w.entries.pop_front();
    if (submitted[i] > 0) {
      const double ratio = static_cast<double>(accepted[i]) / submitted[i];
      c.book.emplace_back(round, spec[i], ratio);  // AcceptanceBook::record
      auto& e = by_s[spec[i]];
      e.first += ratio;
      e.second += 1;
    }
  }
  while (!c.book.empty() && std::get<0>(c.book.front()) <= round - cfg.window_ctx) c.book.pop_front();
  c.rounds = round;  // AdaptiveDrafter::observe_round (drafter.cpp:209-220)
  for (const auto& [s, e] : by_s) {
    const double a = e.first / e.second;
    c.gp.observe(d->index_of(s), t_obs_ms / (s * a + cfg.epsilon), round, cfg.window_ctx);
    auto& lane = c.latency[s];
    lane.emplace_back(round, t_obs_ms);
    while (!lane.empty() && lane.front().first <= round - cfg.window_ctx) lane.pop_front();
  }
  return FASER_OK;
}

faser_status faser_drafter_estimate(faser_drafter* d, const int64_t* req_ids, const int32_t* s, int32_t n,
                                    int32_t b, double r, double* a_hat) {
  if (!d || b < 1 || (n > 0 && (!req_ids || !s || !a_hat))) return FASER_EINVAL;
  const Ctx& c = d->ctx[key_of(b, r)];
  for (int i = 0; i < n; ++i) a_hat[i] = d->estimate(req_ids[i], c, s[i]);
  return FASER_OK;
}

faser_status faser_drafter_request_window(faser_drafter* d, int64_t req_id, const int32_t* qs, int32_t nq,
                                          double* out) {
  if (!d || (nq > 0 && (!qs || !out))) return FASER_EINVAL;
  auto it = d->req.find(req_id);
  for (int j = 0; j < nq; ++j) out[j] = it != d->req.end() ? it->second.rate_for(qs[j]) : -1.0;
  out[nq] = it != d->req.end() ? it->second.overall() : -1.0;
  return FASER_OK;
}

faser_status faser_drafter_release(faser_drafter* d, int64_t req_id) {
  if (!d) return FASER_EINVAL;
  d->req.erase(req_id);
  return FASER_OK;
}

faser_status faser_drafter_posterior(faser_drafter* d, int32_t b, double r, double* mu, double* sigma,
                                     int32_t* rounds) {
  if (!d || b < 1) return FASER_EINVAL;
  auto it = d->ctx.find(key_of(b, r));
  const int m = d->cfg.n_candidates;
  if (it == d->ctx.end()) {
    for (int i = 0; i < m; ++i) {
      if (mu) mu[i] = 0.0;
      if (sigma) sigma[i] = std::sqrt(d->cfg.kernel_var);
    }
    if (rounds) *rounds = 0;
    return FASER_OK;
  }
  Ctx& c = it->second;
  if (c.gp.dirty) c.gp.recompute(d->cfg);
  for (int i = 0; i < m; ++i) {
    if (mu) mu[i] = c.gp.mu[i];
    if (sigma) sigma[i] = c.gp.sigma[i];
  }
  if (rounds) *rounds = c.rounds;
  return FASER_OK;
}

}  // extern "C"

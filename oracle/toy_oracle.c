/* oracle/toy_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C CPU restatement of the reference's
 * toy speculative-decoding path, used as the parity checker for the CUDA engine.
 *
 * Pinned against (a) the reference's own TUs compiled in place (oracle/_ref, see
 * tests/test_oracle.py) and (b) the golden vectors in tests/golden/ (generated from the
 * reference by tests/golden/make_golden.py). Never linked into or called by the product.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/core/{include/specsim,src}/...). Build flags keep x86-64 doubles
 * un-contracted (-ffp-contract=off), matching the reference's Release build. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle.h"

#define GAMMA 0x9e3779b97f4a7c15ull

/* rng.hpp:17-22 */
static uint64_t mix64(uint64_t x) {
  x += GAMMA;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
/* rng.hpp:24-26 */
static uint64_t hash_combine(uint64_t h, uint64_t v) {
  return mix64(h ^ (v + GAMMA + (h << 6) + (h >> 2)));
}
/* rng.hpp:28-32 */
static uint64_t hash_tokens(uint64_t seed, const int32_t* t, int64_t n) {
  uint64_t h = mix64(seed);
  for (int64_t i = 0; i < n; ++i) h = hash_combine(h, (uint64_t)(int64_t)t[i] + 1);
  return h;
}
/* rng.hpp:35-37 */
static double to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
/* rng.hpp:77-79 */
static uint64_t substream(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag)); }

uint64_t oracle_mix64(uint64_t x) { return mix64(x); }
uint64_t oracle_hash_combine(uint64_t h, uint64_t v) { return hash_combine(h, v); }

typedef struct {
  faser_toy_params p;
  uint64_t table_seed, noise_seed, mix_seed;
} toy_t;

/* toylm.cpp:18-26 (constructor seeds + validation) */
static int toy_init(toy_t* m, const faser_toy_params* p) {
  if (p->vocab < 2 || p->layers < 1 || p->order < 1) return FASER_EINVAL;
  if (p->divergence < 0.0 || p->divergence > 1.0) return FASER_EINVAL;
  m->p = *p;
  m->table_seed = substream(p->seed, 0x7461626cull);
  m->noise_seed = substream(p->noise_seed, 0x6e6f6973ull);
  m->mix_seed = substream(p->seed, 0x6d697875ull);
  return FASER_OK;
}

/* toylm.cpp:29-40: hash of the last `order` tokens, front-padded with sentinel V. */
static uint64_t context_hash(const toy_t* m, const int32_t* prefix, int64_t len) {
  uint64_t h = mix64(m->table_seed);
  for (int i = m->p.order; i >= 1; --i) {
    const int64_t tok = (len >= i) ? prefix[len - i] : m->p.vocab;
    h = hash_combine(h, (uint64_t)tok + 1);
  }
  return h;
}

/* toylm.cpp:42-54 */
static void final_and_noise(const toy_t* m, const int32_t* prefix, int64_t len, double* zf,
                            double* zn) {
  const uint64_t ch = context_hash(m, prefix, len);
  const uint64_t nh = hash_tokens(m->noise_seed, prefix, len);
  for (int t = 0; t < m->p.vocab; ++t) {
    if (zf) zf[t] = to_unit(hash_combine(ch, (uint64_t)t + 1)) * m->p.logit_scale;
    if (zn) zn[t] = to_unit(hash_combine(nh, (uint64_t)t + 1)) * m->p.noise_scale;
  }
}

/* toylm.cpp:9-16: strict '>' scan, ties to the lowest id. */
static int argmax_lowest(const double* v, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (v[i] > v[best]) best = i;
  return best;
}

/* toylm.cpp:69-74 */
static int target_next(const toy_t* m, const int32_t* prefix, int64_t len, double* scratch) {
  final_and_noise(m, prefix, len, scratch, NULL);
  return argmax_lowest(scratch, m->p.vocab);
}

/* toylm.cpp:76-85: per-prefix Bernoulli(eta) slip to token 0, else the target argmax. */
static int draft_next(const toy_t* m, const int32_t* prefix, int64_t len, double* scratch) {
  const double u = to_unit(hash_tokens(m->mix_seed, prefix, len));
  if (u < m->p.divergence) return 0;
  return target_next(m, prefix, len, scratch);
}

/* exitctl.cpp:9-17 */
int oracle_k_at(const faser_exit_policy* pol, int layer, int num_layers) {
  if (layer <= pol->l_init || num_layers <= pol->l_init) return pol->k_init;
  if (layer >= num_layers) return pol->k_final;
  const double t = (double)(layer - pol->l_init) / (double)(num_layers - pol->l_init);
  const int k = (int)lround(pol->k_init + (pol->k_final - pol->k_init) * t);
  return k > 1 ? k : 1;
}

/* exitctl.cpp:56-68 */
int oracle_token_exit_test(const double* z, int v, int d, int k) {
  const double ref = z[d];
  int outranking = 0;
  for (int i = 0; i < v; ++i)
    if (z[i] > ref || (z[i] == ref && i < d))
      if (++outranking >= k) return 1;
  return 0;
}

/* ------------------------------------------------------------------ batched row ops */

int oracle_final_and_noise(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                           const int64_t* off, double* zf, double* zn) {
  toy_t m;
  if (toy_init(&m, p)) return FASER_EINVAL;
  for (int i = 0; i < n; ++i) {
    if (off[i + 1] <= off[i]) return FASER_EINVAL;
    final_and_noise(&m, tokens + off[i], off[i + 1] - off[i], zf + (int64_t)i * p->vocab,
                    zn + (int64_t)i * p->vocab);
  }
  return FASER_OK;
}

/* toylm.cpp:56-67 */
int oracle_target_logits(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                         const int64_t* off, const int32_t* layers, double* z) {
  toy_t m;
  if (toy_init(&m, p)) return FASER_EINVAL;
  double* zf = (double*)malloc(sizeof(double) * p->vocab);
  double* zn = (double*)malloc(sizeof(double) * p->vocab);
  int rc = FASER_OK;
  for (int i = 0; i < n && rc == FASER_OK; ++i) {
    const int l = layers[i];
    if (off[i + 1] <= off[i] || l < 1 || l > p->layers) {
      rc = FASER_EINVAL;
      break;
    }
    final_and_noise(&m, tokens + off[i], off[i + 1] - off[i], zf, zn);
    double* out = z + (int64_t)i * p->vocab;
    if (l == p->layers) {
      memcpy(out, zf, sizeof(double) * p->vocab);
    } else {
      const double w = (double)l / (double)p->layers;
      for (int t = 0; t < p->vocab; ++t) out[t] = w * zf[t] + (1.0 - w) * zn[t];
    }
  }
  free(zf);
  free(zn);
  return rc;
}

int oracle_target_next(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                       const int64_t* off, int32_t* out) {
  toy_t m;
  if (toy_init(&m, p)) return FASER_EINVAL;
  double* s = (double*)malloc(sizeof(double) * p->vocab);
  for (int i = 0; i < n; ++i) out[i] = target_next(&m, tokens + off[i], off[i + 1] - off[i], s);
  free(s);
  return FASER_OK;
}

int oracle_draft_next(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                      const int64_t* off, int32_t* out) {
  toy_t m;
  if (toy_init(&m, p)) return FASER_EINVAL;
  double* s = (double*)malloc(sizeof(double) * p->vocab);
  for (int i = 0; i < n; ++i) out[i] = draft_next(&m, tokens + off[i], off[i + 1] - off[i], s);
  free(s);
  return FASER_OK;
}

/* toylm.cpp:87-101 */
int oracle_autoregressive_decode(const faser_toy_params* p, const int32_t* prompt, int32_t len,
                                 int32_t max_out, int32_t* out, int32_t* n_out) {
  toy_t m;
  if (toy_init(&m, p) || len < 1 || max_out < 0) return FASER_EINVAL;
  int32_t* seq = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len + max_out + 1));
  double* s = (double*)malloc(sizeof(double) * p->vocab);
  memcpy(seq, prompt, sizeof(int32_t) * len);
  int64_t L = len;
  int n = 0;
  while (n < max_out) {
    const int tok = target_next(&m, seq, L, s);
    out[n++] = tok;
    seq[L++] = tok;
    if (tok == p->vocab - 1) break;
  }
  *n_out = n;
  free(seq);
  free(s);
  return FASER_OK;
}

/* ------------------------------------------------------------------ engine semantics */

/* sdcore.cpp:45-59 over context ctx[0..len); ctx must have room for s more tokens. */
static int draft_tokens(const toy_t* m, int32_t* ctx, int64_t len, int s, int remaining,
                        int32_t* out, double* scratch) {
  const int budget = s < remaining ? s : remaining;
  int n = 0;
  for (int i = 0; i < budget; ++i) {
    const int tok = draft_next(m, ctx, len + i, scratch);
    out[n++] = tok;
    ctx[len + i] = tok;
    if (tok == m->p.vocab - 1) break;
  }
  return n;
}

/* sdcore.cpp:61-81 */
static void full_verify(const toy_t* m, int32_t* ctx, int64_t len, const int32_t* d, int count,
                        faser_verify_outcome* o, double* scratch) {
  memset(o, 0, sizeof(*o));
  o->base_len = len;
  o->submitted = count;
  o->full_layers_run = (double)m->p.layers * count;
  o->recovery_token = -1;
  o->pruned_index = o->pruned_layer = -1;
  for (int j = 0; j < count; ++j) {
    const int truth = target_next(m, ctx, len + j, scratch);
    if (d[j] == truth) {
      ++o->accepted_count;
      ctx[len + j] = d[j];
    } else {
      o->has_recovery = 1;
      o->recovery_token = truth;
      break;
    }
  }
}

/* sdcore.cpp:83-180. k_table (nullable) replaces ExitPolicy::k_at. ctx has room for count. */
static void verify_ee(const toy_t* m, int32_t* ctx, int64_t len, int committed_len, int exempt,
                      const int32_t* d, int count, const faser_exit_policy* pol,
                      const int32_t* k_table, const faser_gate_plan* gate,
                      faser_verify_outcome* o) {
  const int V = m->p.vocab, L = m->p.layers;
  double* zf = (double*)malloc(sizeof(double) * V * count);
  double* zn = (double*)malloc(sizeof(double) * V * count);
  double* z = (double*)malloc(sizeof(double) * V);
  int prune_layer[FASER_MAX_SPEC];
  memset(o, 0, sizeof(*o));
  o->base_len = len;
  o->submitted = count;
  o->recovery_token = -1;
  o->pruned_index = o->pruned_layer = -1;
  /* position j is conditioned on ctx ++ d[0..j) (sdcore.cpp:96-105) */
  for (int j = 0; j < count; ++j) ctx[len + j] = d[j];
  for (int j = 0; j < count; ++j) final_and_noise(m, ctx, len + j, zf + j * V, zn + j * V);

  int active = count;
  for (int j = 0; j < count; ++j) prune_layer[j] = L;
  if (gate->first_layer < gate->stop_layer) {
    const int last = gate->stop_layer < L ? gate->stop_layer : L;
    for (int layer = gate->first_layer > 1 ? gate->first_layer : 1; layer < last && active > 0;
         ++layer) {
      ++o->gate_layers;
      const int k = k_table ? k_table[layer] : oracle_k_at(pol, layer, L);
      const double w = (double)layer / L;
      for (int j = 0; j < active; ++j) {
        if (committed_len + j == exempt) continue;
        for (int v = 0; v < V; ++v) z[v] = w * zf[j * V + v] + (1.0 - w) * zn[j * V + v];
        if (oracle_token_exit_test(z, V, d[j], k)) {
          for (int jj = j; jj < active; ++jj) prune_layer[jj] = layer;
          active = j;
          o->has_pruned = 1;
          o->pruned_index = j;
          o->pruned_layer = layer;
          o->prune_layers[o->n_prune_layers++] = layer;
          break;
        }
      }
    }
  }
  int mismatch = 0;
  for (int j = 0; j < active; ++j) {
    const int truth = argmax_lowest(zf + j * V, V);
    if (d[j] == truth) {
      ++o->accepted_count;
    } else {
      o->has_recovery = 1;
      o->recovery_token = truth;
      mismatch = 1;
      break;
    }
  }
  if (active == 0) { /* force-verify token 0 (sdcore.cpp:150-166) */
    const int truth = argmax_lowest(zf, V);
    if (d[0] == truth) {
      o->accepted_count = 1;
    } else {
      o->has_recovery = 1;
      o->recovery_token = truth;
      mismatch = 1;
    }
    if (count > 1) {
      o->has_pruned = 1;
      o->pruned_index = 1;
      o->pruned_layer = prune_layer[1];
    } else {
      o->has_pruned = 0;
      o->pruned_index = o->pruned_layer = -1;
    }
    active = 1;
  }
  for (int j = 0; j < count; ++j) o->full_layers_run += (j < active) ? L : prune_layer[j];
  /* false-prune bookkeeping (sdcore.cpp:171-178): target argmax at the cut position */
  if (o->has_pruned && !mismatch && o->accepted_count == o->pruned_index) {
    const int cut = o->pruned_index;
    if (cut < count) o->false_prune = (d[cut] == argmax_lowest(zf + cut * V, V));
  }
  free(zf);
  free(zn);
  free(z);
}

int oracle_draft_tokens(const faser_toy_params* p, int32_t n, const int32_t* tokens,
                        const int64_t* off, const int32_t* s, const int32_t* remaining,
                        int32_t* out, int32_t* out_len) {
  toy_t m;
  if (toy_init(&m, p)) return FASER_EINVAL;
  double* sc = (double*)malloc(sizeof(double) * p->vocab);
  int rc = FASER_OK;
  for (int i = 0; i < n; ++i) {
    if (remaining[i] <= 0) { rc = FASER_EILLEGAL_STATE; break; }
    if (s[i] < 1) { rc = FASER_EINVAL; break; }
    const int64_t len = off[i + 1] - off[i];
    int32_t* ctx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len + s[i]));
    memcpy(ctx, tokens + off[i], sizeof(int32_t) * len);
    out_len[i] = draft_tokens(&m, ctx, len, s[i], remaining[i], out + (int64_t)i * FASER_MAX_SPEC, sc);
    free(ctx);
  }
  free(sc);
  return rc;
}

int oracle_verify(const faser_toy_params* p, int32_t n, const int32_t* tokens, const int64_t* off,
                  const int32_t* committed_len, const int32_t* exempt, const int32_t* drafted,
                  const int32_t* drafted_len, const faser_exit_policy* policy,
                  const faser_gate_plan* gate, const int32_t* k_table, faser_verify_outcome* out) {
  toy_t m;
  if (toy_init(&m, p)) return FASER_EINVAL;
  double* sc = (double*)malloc(sizeof(double) * p->vocab);
  for (int i = 0; i < n; ++i) {
    const int64_t len = off[i + 1] - off[i];
    const int count = drafted_len[i];
    int32_t* ctx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len + count));
    memcpy(ctx, tokens + off[i], sizeof(int32_t) * len);
    const int32_t* d = drafted + (int64_t)i * FASER_MAX_SPEC;
    if (gate == NULL)
      full_verify(&m, ctx, len, d, count, out + i, sc);
    else
      verify_ee(&m, ctx, len, committed_len[i], exempt ? exempt[i] : -1, d, count, policy, k_table,
                gate, out + i);
    free(ctx);
  }
  free(sc);
  return FASER_OK;
}

/* workload.cpp:116-122 + rng.hpp:41-70 (SplitMixStream::next_int, modulo) */
int oracle_synth_prompt(uint64_t seed, int32_t index, int32_t len, int32_t vocab, int32_t* out) {
  const int n = len > 1 ? len : 1;
  uint64_t state = mix64(substream(substream(seed, 0x70726d70ull), (uint64_t)(int64_t)index));
  const uint64_t span = (uint64_t)(vocab - 2 - 0) + 1;
  for (int i = 0; i < n; ++i) {
    state += GAMMA;
    out[i] = (int32_t)(mix64(state) % span);
  }
  return FASER_OK;
}

/* The lens substream of synth_workload (workload.cpp:73-98): for a backlog (all arrivals at
 * t=0) record i draws input_len then output_len from substream(seed,"lens"). */
int oracle_backlog_lengths(uint64_t seed, int32_t n, int32_t in_lo, int32_t in_hi, int32_t out_lo,
                           int32_t out_hi, int32_t* in_len, int32_t* out_len) {
  uint64_t state = mix64(substream(seed, 0x6c656e73ull));
  for (int i = 0; i < n; ++i) {
    state += GAMMA;
    in_len[i] = in_lo + (int32_t)(mix64(state) % ((uint64_t)(in_hi - in_lo) + 1));
    state += GAMMA;
    out_len[i] = out_lo + (int32_t)(mix64(state) % ((uint64_t)(out_hi - out_lo) + 1));
  }
  return FASER_OK;
}

/* Same schedule as specref_sched_k (ref_shim.cpp). */
int32_t oracle_sched_k(uint64_t seed, int64_t req_id, int32_t round) {
  static const int kS[8] = {1, 2, 3, 4, 5, 6, 8, 10};
  const uint64_t h = hash_combine(hash_combine(mix64(seed), (uint64_t)req_id + 1), (uint64_t)round + 1);
  return kS[h % 8];
}

/* sdcore.cpp:182-197 applied to a flat request. Returns tokens committed. */
static int commit(const toy_t* m, int32_t* committed, int* n_committed, int max_out, int* done,
                  const faser_verify_outcome* o, const int32_t* d) {
  int c = 0;
  for (int j = 0; j < o->accepted_count && !*done; ++j) {
    committed[(*n_committed)++] = d[j];
    ++c;
    if (d[j] == m->p.vocab - 1 || *n_committed == max_out) *done = 1;
  }
  if (o->has_recovery && !*done) {
    committed[(*n_committed)++] = o->recovery_token;
    ++c;
    if (o->recovery_token == m->p.vocab - 1 || *n_committed == max_out) *done = 1;
  }
  return c;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* Single-threaded serving loop; identical semantics to specref_run_episode. */
int oracle_run_episode(const specref_episode_cfg* cfg, const int32_t* prompt_tokens,
                       const int64_t* prompt_off, const int32_t* max_out, int32_t* out_tokens,
                       int32_t out_cap, int32_t* out_len, faser_round_result* round_log,
                       int64_t log_cap, int64_t* n_log, specref_episode_stats* stats) {
  toy_t m;
  if (toy_init(&m, &cfg->model)) return FASER_EINVAL;
  const int n = cfg->n_requests;
  int64_t max_ctx = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t c = prompt_off[i + 1] - prompt_off[i] + max_out[i] + FASER_MAX_SPEC + 1;
    if (c > max_ctx) max_ctx = c;
  }
  int32_t* ctx = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_ctx);
  int32_t* comm = (int32_t*)calloc((size_t)n * (size_t)(out_cap + FASER_MAX_SPEC + 1), sizeof(int32_t));
  int* ncomm = (int*)calloc(n, sizeof(int));
  int* done = (int*)calloc(n, sizeof(int));
  int* exempt = (int*)malloc(sizeof(int) * n);
  int* rounds = (int*)calloc(n, sizeof(int));
  double* t_first = (double*)malloc(sizeof(double) * n);
  double* t_last = (double*)malloc(sizeof(double) * n);
  int* live = (int*)malloc(sizeof(int) * (n + 1));
  double* sc = (double*)malloc(sizeof(double) * cfg->model.vocab);
  const int stride = out_cap + FASER_MAX_SPEC + 1;
  for (int i = 0; i < n; ++i) {
    exempt[i] = -1;
    t_first[i] = t_last[i] = -1.0;
    done[i] = max_out[i] <= 0;
  }
  specref_episode_stats st;
  memset(&st, 0, sizeof(st));
  int n_live = 0, next = 0;
  int64_t logged = 0;
  const double t0 = now_s();
  int64_t round = 0;
  for (;;) {
    while (next < n && n_live < cfg->max_batch) {
      if (!done[next]) live[n_live++] = next;
      ++next;
    }
    if (n_live == 0) break;
    if (cfg->max_rounds > 0 && round >= cfg->max_rounds) break;
    int keep = 0;
    const double t_round = 0; (void)t_round;
    faser_round_result rr;
    for (int pos = 0; pos < n_live; ++pos) {
      const int id = live[pos];
      const int64_t plen = prompt_off[id + 1] - prompt_off[id];
      memcpy(ctx, prompt_tokens + prompt_off[id], sizeof(int32_t) * plen);
      memcpy(ctx + plen, comm + (int64_t)id * stride, sizeof(int32_t) * ncomm[id]);
      const int64_t len = plen + ncomm[id];
      const int k = cfg->k_mode == 1 ? oracle_sched_k(cfg->k_seed, id, rounds[id]) : cfg->fixed_k;
      memset(&rr, 0, sizeof(rr));
      rr.req_id = id;
      rr.spec_length = k;
      int32_t d[FASER_MAX_SPEC];
      rr.drafted = draft_tokens(&m, ctx, len, k, max_out[id] - ncomm[id], d, sc);
      if (cfg->early_exit)
        verify_ee(&m, ctx, len, ncomm[id], exempt[id], d, rr.drafted, &cfg->policy, NULL, &cfg->gate,
                  &rr.outcome);
      else
        full_verify(&m, ctx, len, d, rr.drafted, &rr.outcome, sc);
      const int before = ncomm[id];
      rr.committed = commit(&m, comm + (int64_t)id * stride, &ncomm[id], max_out[id], &done[id],
                            &rr.outcome, d);
      for (int j = 0; j < rr.committed; ++j) rr.tokens[j] = comm[(int64_t)id * stride + before + j];
      if (cfg->exempt_rule) exempt[id] = rr.outcome.has_pruned ? before + rr.outcome.pruned_index : -1;
      rr.done = done[id];
      rr.exempt_position = exempt[id];
      rr.n_committed_total = ncomm[id];
      rounds[id] += 1;
      st.drafted += rr.drafted;
      st.submitted += rr.outcome.submitted;
      st.accepted += rr.outcome.accepted_count;
      st.committed += rr.committed;
      st.false_prunes += rr.outcome.false_prune;
      st.layer_work += rr.outcome.full_layers_run;
      st.layer_work_full += (double)cfg->model.layers * rr.outcome.submitted;
      if (round_log && logged < log_cap) round_log[logged] = rr;
      ++logged;
    }
    const double now_ms = (now_s() - t0) * 1e3;
    for (int pos = 0; pos < n_live; ++pos) {
      const int id = live[pos];
      if (t_first[id] < 0 && ncomm[id] > 0) t_first[id] = now_ms;
      t_last[id] = now_ms;
      if (!done[id]) live[keep++] = id;
    }
    n_live = keep;
    ++round;
  }
  st.wall_s = now_s() - t0;
  st.rounds = round;
  double* tp = (double*)malloc(sizeof(double) * (n + 1));
  int ntp = 0;
  for (int i = 0; i < n; ++i) {
    out_len[i] = ncomm[i];
    for (int j = 0; j < ncomm[i] && j < out_cap; ++j)
      out_tokens[(int64_t)i * out_cap + j] = comm[(int64_t)i * stride + j];
    if (done[i]) ++st.finished;
    if (ncomm[i] >= 2 && t_first[i] >= 0) tp[ntp++] = (t_last[i] - t_first[i]) / (ncomm[i] - 1);
  }
  if (ntp) {
    qsort(tp, ntp, sizeof(double), cmp_double);
    st.p50_tpot_ms = tp[ntp / 2];
    double s = 0;
    for (int i = 0; i < ntp; ++i) s += tp[i];
    st.mean_tpot_ms = s / ntp;
  }
  if (n_log) *n_log = logged;
  if (stats) *stats = st;
  free(tp); free(ctx); free(comm); free(ncomm); free(done); free(exempt); free(rounds);
  free(t_first); free(t_last); free(live); free(sc);
  return FASER_OK;
}

/* oracle/oracle.h — TEST INFRASTRUCTURE ONLY. Shared declarations of the CPU oracle:
 * the reference TUs wrapped by ref_shim.cpp (libspecsim_ref.so, symbols specref_*) and the
 * plain-C restatement toy_oracle.c (liboracle.so, symbols oracle_*). Both take the same
 * structs so tests can cross-check them against each other and against the CUDA engine. */
#ifndef FASER_ORACLE_H
#define FASER_ORACLE_H
#include <stdint.h>
#include "faser/engine.h"
#ifdef __cplusplus
extern "C" {
#endif

typedef struct specref_episode_cfg {
  faser_toy_params model;
  int32_t n_requests;
  int32_t max_batch;
  int32_t early_exit;   // 0: full_verify, 1: verify_with_early_exit with `gate`
  int32_t k_mode;       // 0: fixed_k, 1: specref_sched_k(k_seed, ...)
  int32_t fixed_k;
  int32_t exempt_rule;  // 1: exempt = committed_before + pruned_at.first for one round
  int32_t threads;      // persistent worker pool size (>= 1)
  int32_t max_rounds;   // 0: run to completion
  uint64_t k_seed;
  faser_exit_policy policy;
  faser_gate_plan gate;
} specref_episode_cfg;

typedef struct specref_episode_stats {
  int64_t rounds;
  int64_t drafted;
  int64_t submitted;
  int64_t accepted;
  int64_t committed;
  int64_t false_prunes;
  int64_t finished;
  double layer_work;
  double layer_work_full;
  double wall_s;
  double p50_tpot_ms;
  double mean_tpot_ms;
} specref_episode_stats;

#ifdef __cplusplus
}
#endif
#endif

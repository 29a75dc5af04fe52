"""ctypes mirror of include/faser/engine.h (the C ABI of the CUDA engine).

Struct layouts here must match the header byte for byte; tests/test_abi.py checks sizes
against the values the library itself reports.
"""
import ctypes as C

MAX_SPEC = 32
MAX_LAYERS = 128

OK, EINVAL, EILLEGAL_STATE, ECONFIG, EPARSE, EFIT, ECUDA, ENCCL, ENOMEM, ECAPACITY = range(10)
STATUS_NAMES = {
    0: "OK", 1: "EINVAL", 2: "EILLEGAL_STATE", 3: "ECONFIG", 4: "EPARSE", 5: "EFIT",
    6: "ECUDA", 7: "ENCCL", 8: "ENOMEM", 9: "ECAPACITY",
}
MODEL_TOY, MODEL_LLAMA = 0, 1
MODE_VSD, MODE_VSD_AD, MODE_VSD_AD_EE, MODE_FULL = range(4)


class ToyParams(C.Structure):
    """LayeredToyLM::Params (toylm.hpp:42-51); defaults = config.hpp:41 (seed 1, eta 0.3)."""
    _fields_ = [
        ("seed", C.c_uint64), ("vocab", C.c_int32), ("layers", C.c_int32),
        ("order", C.c_int32), ("reserved0", C.c_int32), ("divergence", C.c_double),
        ("noise_seed", C.c_uint64), ("logit_scale", C.c_double), ("noise_scale", C.c_double),
    ]

    @classmethod
    def default(cls, divergence=0.3, **kw):
        p = cls(seed=1, vocab=64, layers=32, order=2, divergence=divergence, noise_seed=2,
                logit_scale=4.0, noise_scale=1.0)
        for k, v in kw.items():
            setattr(p, k, v)
        return p


class ExitPolicy(C.Structure):
    _fields_ = [("l_init", C.c_int32), ("k_init", C.c_int32), ("k_final", C.c_int32)]

    @classmethod
    def default(cls):
        return cls(8, 10, 2)


class GatePlan(C.Structure):
    _fields_ = [("first_layer", C.c_int32), ("stop_layer", C.c_int32), ("s_eff", C.c_double)]


class GateEntry(C.Structure):
    _fields_ = [("spec_length", C.c_int32), ("reserved0", C.c_int32),
                ("accept_estimate", C.c_double)]


class OverlapPlan(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("chunk", C.c_int32), ("r", C.c_double),
                ("predicted_ms", C.c_double), ("serial_ms", C.c_double)]


class LatencyParams(C.Structure):
    _fields_ = [("stage", C.c_int32), ("reserved0", C.c_int32)] + [
        (n, C.c_double) for n in ("knee", "a1", "gamma1", "a2", "gamma2", "c0", "c1", "c2")]


class LatencyModel(C.Structure):
    _fields_ = [("draft", LatencyParams), ("target", LatencyParams),
                ("ee_check", LatencyParams), ("prune", LatencyParams)]


class VerifyOutcome(C.Structure):
    _fields_ = [
        ("submitted", C.c_int32), ("accepted_count", C.c_int32), ("has_recovery", C.c_int32),
        ("recovery_token", C.c_int32), ("has_pruned", C.c_int32), ("pruned_index", C.c_int32),
        ("pruned_layer", C.c_int32), ("gate_layers", C.c_int32), ("full_layers_run", C.c_double),
        ("false_prune", C.c_int32), ("n_prune_layers", C.c_int32),
        ("prune_layers", C.c_int32 * MAX_SPEC), ("base_len", C.c_int64),
    ]

    def as_tuple(self):
        return (self.submitted, self.accepted_count, self.has_recovery,
                self.recovery_token if self.has_recovery else -1, self.has_pruned,
                self.pruned_index if self.has_pruned else -1,
                self.pruned_layer if self.has_pruned else -1, self.gate_layers,
                self.full_layers_run, self.false_prune,
                tuple(self.prune_layers[:self.n_prune_layers]), self.base_len)


class LlamaShape(C.Structure):
    """faser_llama_shape: Llama-style random-init bf16 model (configs 3-5)."""
    _fields_ = [(n, C.c_int32) for n in ("d_model", "layers", "n_heads", "n_kv_heads", "head_dim",
                                         "ffn", "vocab", "reserved0")] + [
        (n, C.c_double) for n in ("rope_theta", "rms_eps", "bigram_scale", "embed_noise",
                                  "init_std", "hard_fraction")] + [("seed", C.c_uint64)]


class ModelDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved0", C.c_int32), ("toy", ToyParams),
                ("draft", LlamaShape), ("target", LlamaShape), ("bigram_a", C.c_uint32),
                ("bigram_b", C.c_uint32)]


class EngineCfg(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("max_batch", C.c_int32), ("max_seq_len", C.c_int32),
        ("mode", C.c_int32), ("default_spec_length", C.c_int32), ("exempt_rule", C.c_int32),
        ("exit_policy", ExitPolicy), ("max_pending", C.c_int32), ("pending_tokens", C.c_int32),
        ("max_spec_length", C.c_int32), ("prefill_rows", C.c_int32), ("debug_capture", C.c_int32),
        ("prefill_lane", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32), ("tp_group", C.c_void_p),
    ]


class StepPlan(C.Structure):
    _fields_ = [("gate", GatePlan), ("use_k_table", C.c_int32),
                ("k_table", C.c_int32 * (MAX_LAYERS + 1)), ("overlap", OverlapPlan),
                ("lane_mode", C.c_int32), ("reserved_lane", C.c_int32)]


LANES_OVERLAP, LANES_ISOLATED = 0, 1
EV_DRAFT_CHUNK, EV_VERIFY_CHUNK, EV_RESET, EV_COMMIT = 0, 1, 2, 3


class TimelineEvent(C.Structure):
    """TimelineEvent (overlap.hpp:29-34), measured on the lanes."""
    _fields_ = [("kind", C.c_int32), ("chunk", C.c_int32), ("start_ms", C.c_double), ("end_ms", C.c_double)]


class TimelineInfo(C.Structure):
    """PipelineTimeline totals (overlap.hpp:49-56) + the partitions and the frontier per chunk."""
    _fields_ = [("n_events", C.c_int32), ("n_chunks", C.c_int32), ("draft_sms", C.c_int32),
                ("verify_sms", C.c_int32), ("green", C.c_int32), ("cancelled_draft_steps", C.c_int32),
                ("lane_mode", C.c_int32), ("survivors", C.c_int32),
                ("chunk_alive", C.c_int32 * (MAX_SPEC + 1)), ("chunk_rows", C.c_int32 * (MAX_SPEC + 1)),
                ("chunk_resets", C.c_int32 * (MAX_SPEC + 1)), ("reserved0", C.c_int32),
                ("makespan_ms", C.c_double), ("draft_busy_ms", C.c_double), ("verify_busy_ms", C.c_double),
                ("wasted_draft_ms", C.c_double)]


class RoundResult(C.Structure):
    _fields_ = [
        ("req_id", C.c_int64), ("spec_length", C.c_int32), ("drafted", C.c_int32),
        ("outcome", VerifyOutcome), ("committed", C.c_int32), ("done", C.c_int32),
        ("exempt_position", C.c_int32), ("n_committed_total", C.c_int32),
        ("tokens", C.c_int32 * (MAX_SPEC + 1)),
    ]

    def as_tuple(self):
        return (self.req_id, self.spec_length, self.drafted, self.outcome.as_tuple(),
                self.committed, self.done, self.exempt_position, self.n_committed_total,
                tuple(self.tokens[:self.committed]))


class EpisodeCfg(C.Structure):
    """specref_episode_cfg (oracle/oracle.h) — used only by tests / bench baselines."""
    _fields_ = [
        ("model", ToyParams), ("n_requests", C.c_int32), ("max_batch", C.c_int32),
        ("early_exit", C.c_int32), ("k_mode", C.c_int32), ("fixed_k", C.c_int32),
        ("exempt_rule", C.c_int32), ("threads", C.c_int32), ("max_rounds", C.c_int32),
        ("k_seed", C.c_uint64), ("policy", ExitPolicy), ("gate", GatePlan),
    ]


class EpisodeStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("rounds", "drafted", "submitted", "accepted", "committed",
                                         "false_prunes", "finished")] + [
        (n, C.c_double) for n in ("layer_work", "layer_work_full", "wall_s", "p50_tpot_ms",
                                  "mean_tpot_ms")]


# -------------------------------------------------------------------- shared helpers
S_CANDIDATES = (1, 2, 3, 4, 5, 6, 8, 10)  # DrafterConfig::candidates, drafter.hpp:16
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


def mix64(x):
    """rng.hpp:17-22 (Python ints, masked to 64 bits)."""
    x = (x + _GAMMA) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def hash_combine(h, v):
    """rng.hpp:24-26."""
    return mix64(h ^ ((v + _GAMMA + (h << 6) + (h >> 2)) & _M64))


def sched_k(seed, req_id, rnd):
    """Seeded per-request speculative length over S for bit-exact dynamic-k runs
    (same as specref_sched_k in oracle/ref_shim.cpp)."""
    h = hash_combine(hash_combine(mix64(seed), (req_id + 1) & _M64), rnd + 1)
    return S_CANDIDATES[h % 8]

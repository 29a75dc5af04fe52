"""Llama-style draft/target presets (configs 3-5) and a ModelDesc builder.

The reference has no transformer; these are random-init bf16 models of
the shapes BASELINE.json names. Acceptance is tunable through the bigram construction
(embedding(t) = bigram_scale * W_lm[g(t)] + noise, g(t) = (a*t + b) mod V), the analogue of
LayeredToyLM's divergence eta (toylm.cpp:76-85); see DESIGN.md.
"""
from . import abi

BIGRAM_A = 7919  # prime, coprime to every preset vocab


def shape(d, layers, heads, kv_heads, head_dim, ffn, vocab, seed, theta=10000.0, eps=1e-5,
          bigram=8.0, noise=0.02, std=0.02, hard=0.0):
    return abi.LlamaShape(d_model=d, layers=layers, n_heads=heads, n_kv_heads=kv_heads,
                          head_dim=head_dim, ffn=ffn, vocab=vocab, reserved0=0, rope_theta=theta,
                          rms_eps=eps, bigram_scale=bigram, embed_noise=noise, init_std=std,
                          hard_fraction=hard, seed=seed)


def _pair(draft, target, b=12345):
    return abi.ModelDesc(kind=abi.MODEL_LLAMA, reserved0=0, toy=abi.ToyParams.default(),
                         draft=draft, target=target, bigram_a=BIGRAM_A,
                         bigram_b=b % target.vocab)


# Target bigram strength + hard-token fraction set the acceptance rate (tuned on B200,
# DESIGN.md section 3): a strong bigram makes the target follow its successor map; the draft
# disagrees exactly on the target's "hard" tokens (successor shifted by V/2).
TARGET_BIGRAM = {"tiny": 2.0, "cfg3": 32.0, "cfg4": 128.0}
TARGET_HARD = {"tiny": 0.0, "cfg3": 0.2, "cfg4": 0.2}
DRAFT_BIGRAM = 24.0


def config3(target_bigram=None, draft_bigram=None, hard=None):
    """llama-68m-shaped draft / TinyLlama-1.1B-shaped target, V=32000 (config 3)."""
    tb = TARGET_BIGRAM["cfg3"] if target_bigram is None else target_bigram
    db = DRAFT_BIGRAM if draft_bigram is None else draft_bigram
    hf = TARGET_HARD["cfg3"] if hard is None else hard
    return _pair(shape(768, 2, 12, 12, 64, 3072, 32000, seed=11, bigram=db),
                 shape(2048, 22, 32, 4, 64, 5632, 32000, seed=12, bigram=tb, hard=hf))


def config4(target_bigram=None, draft_bigram=None, hard=None):
    """Llama-3.2-1B-shaped draft / Llama-3.1-8B-shaped target, V=128256 (config 4)."""
    tb = TARGET_BIGRAM["cfg4"] if target_bigram is None else target_bigram
    db = DRAFT_BIGRAM if draft_bigram is None else draft_bigram
    hf = TARGET_HARD["cfg4"] if hard is None else hard
    return _pair(shape(2048, 16, 32, 8, 64, 8192, 128256, seed=21, theta=500000.0, bigram=db),
                 shape(4096, 32, 32, 8, 128, 14336, 128256, seed=22, theta=500000.0, bigram=tb, hard=hf))


def tiny(target_bigram=None, draft_bigram=None, vocab=512, hard=None):
    """Small pair with the same structure (GQA target, MHA draft) for fast parity tests."""
    tb = TARGET_BIGRAM["tiny"] if target_bigram is None else target_bigram
    db = DRAFT_BIGRAM if draft_bigram is None else draft_bigram
    hf = TARGET_HARD["tiny"] if hard is None else hard
    return _pair(shape(128, 2, 2, 2, 64, 256, vocab, seed=31, bigram=db),
                 shape(256, 4, 4, 2, 64, 512, vocab, seed=32, bigram=tb, hard=hf))


def config5(target_bigram=None, draft_bigram=None, hard=None):
    """Llama-3.2-1B-shaped draft / Llama-3.1-70B-shaped target (d8192, L80, 64q/8kv x 128,
    FFN 28672), V=128256 (config 5: TP=8 verification, ~17.4 GB of target weights per rank)."""
    tb = TARGET_BIGRAM["cfg4"] if target_bigram is None else target_bigram
    db = DRAFT_BIGRAM if draft_bigram is None else draft_bigram
    hf = TARGET_HARD["cfg4"] if hard is None else hard
    return _pair(shape(2048, 16, 32, 8, 64, 8192, 128256, seed=21, theta=500000.0, bigram=db),
                 shape(8192, 80, 64, 8, 128, 28672, 128256, seed=52, theta=500000.0, bigram=tb, hard=hf))


def tp_tiny(target_bigram=None, draft_bigram=None, hard=None):
    """Small pair whose target splits over 1/2/4/8 tensor-parallel ranks (16q/8kv heads, FFN 512,
    V 1024) for the TP parity tests."""
    tb = TARGET_BIGRAM["tiny"] if target_bigram is None else target_bigram
    db = DRAFT_BIGRAM if draft_bigram is None else draft_bigram
    hf = 0.0 if hard is None else hard
    return _pair(shape(128, 2, 2, 2, 64, 256, 1024, seed=41, bigram=db),
                 shape(256, 3, 16, 8, 64, 512, 1024, seed=42, bigram=tb, hard=hf))


def tiny128(target_bigram=None, draft_bigram=None, hard=None):
    """Small pair with the config-4/5 head geometry (head_dim 128, GQA 4, theta 5e5, tied-style
    MHA draft with head_dim 64) for lossless parity tests of the hd-128 paths."""
    tb = TARGET_BIGRAM["tiny"] if target_bigram is None else target_bigram
    db = DRAFT_BIGRAM if draft_bigram is None else draft_bigram
    hf = 0.0 if hard is None else hard
    return _pair(shape(256, 2, 4, 4, 64, 512, 2048, seed=61, theta=500000.0, bigram=db),
                 shape(512, 3, 8, 2, 128, 1024, 2048, seed=62, theta=500000.0, bigram=tb, hard=hf))


PRESETS = {"tiny": tiny, "cfg3": config3, "cfg4": config4, "cfg5": config5, "tp_tiny": tp_tiny, "tiny128": tiny128}


def fitted_latency_model(path=None, share_path=None):
    """abi.LatencyModel from the B200 stage-latency fits: ee_check / prune from
    tools/profile_latency.py (profiles/r01_latency_model.json), draft / target with their measured
    SM-share factor from tools/lane_profile.py (profiles/r02_lane_profile.json: green-context
    partitions at r in {0.25, 0.5, 0.75} + whole-GPU samples) when present. None when absent."""
    import json
    import os
    prof = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    path = path or os.path.join(prof, "r01_latency_model.json")
    share_path = share_path or os.path.join(prof, "r02_lane_profile.json")
    if not os.path.exists(path):
        return None
    m = dict(json.load(open(path))["model"])
    if os.path.exists(share_path):
        m.update(json.load(open(share_path))["model"])
    out = abi.LatencyModel()
    for name in ("draft", "target", "ee_check", "prune"):
        p = getattr(out, name)
        for k, v in m[name].items():
            setattr(p, k, int(v) if k == "stage" else float(v))
    return out

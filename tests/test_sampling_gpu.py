"""GPU tier: sampling acceptance (faser_set_sampling; north-star K6 "greedy/rejection-sampling",
beyond the reference, which is greedy only: SPEC.md:8).

The draft and target LM heads sample with coupled Gumbel-max noise keyed by (seed, request id,
absolute position) and K5 accepts drafted tokens while they equal the target's sample. Checked
here: every committed sequence equals autoregressive coupled-Gumbel sampling from the fp32
target oracle (oracle/sampling.py) — lossless, and independent of the drafter's k_i — with any
divergence explained by a near-tie of the perturbed target row within the bf16 logit tolerance;
sampling is active (outputs differ from greedy) and speculation still pays (drafted tokens are
accepted)."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import lmoracle
from oracle import sampling as S
from paper_2604_20503_b200 import abi, engine, llama

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-2  # bf16 vs the fp32 oracle, relative to the row's logit range (north star)


@pytest.fixture(autouse=True)
def _gpu():
    if not has_gpu():
        pytest.skip("no GPU")


def run(desc, prompts, max_out, tau, seed, kpat, mode=abi.MODE_VSD, rid0=1000, gate=None, stats=None, **kw):
    eng = engine.ServingEngine(desc=desc, max_batch=4, max_seq_len=160, mode=mode, default_spec_length=4,
                               max_spec_length=16, prefill_rows=1024, **kw)
    eng.set_sampling(tau, seed)
    for i, (p, m) in enumerate(zip(prompts, max_out)):
        eng.submit(rid0 + i, p, m)
    acc = sub = s = 0
    while eng.live_requests():
        live = eng.live_requests()
        eng.set_spec_lengths(live, [kpat(r, s) for r in live])
        if gate is not None:
            eng.set_gate(gate)
        for r in eng.step():
            acc += r.outcome.accepted_count
            sub += r.outcome.submitted
            if stats is not None:
                stats["pruned"] = stats.get("pruned", 0) + r.outcome.has_pruned
        s += 1
    out = [eng.committed(rid0 + i) for i in range(len(prompts))]
    eng.close()
    return out, acc, sub


def check_vs_oracle(desc, prompts, max_out, got, tau, seed):
    V = desc.target.vocab
    tgt = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b)
    exact = differs_from_greedy = 0
    for i, (p, m) in enumerate(zip(prompts, max_out)):
        ref, rows = S.sampled_decode(tgt, p, m, V - 1, 1000 + i, seed, tau)
        differs_from_greedy += ref != tgt.greedy(p, m, V - 1)
        if got[i] == ref:
            exact += 1
            continue
        j = next((q for q in range(min(len(got[i]), len(ref))) if got[i][q] != ref[q]), None)
        assert j is not None, (i, got[i], ref)  # one is a prefix of the other: EOS / length bug
        z, y = rows[j]
        ys = np.sort(y)
        # bf16 logits move each perturbed entry by <= LOGIT_TOL * range(z) / tau
        assert ys[-1] - ys[-2] <= 2 * LOGIT_TOL * (z.max() - z.min()) / tau, (i, j, ys[-1] - ys[-2])
    tgt.close()
    return exact, differs_from_greedy


KPATS = {"k1": lambda r, s: 1, "k4": lambda r, s: 4, "cycle": lambda r, s: (1, 2, 3, 4, 5, 6, 8, 10)[(r + s) % 8]}


@pytest.mark.parametrize("preset,tau", [("tiny", 1.0), ("tiny", 0.5), ("tiny128", 1.0)])
@pytest.mark.parametrize("kpat", ["k1", "k4", "cycle"])
def test_sampling_lossless_vs_oracle(preset, tau, kpat):
    desc = llama.PRESETS[preset]()
    V = desc.target.vocab
    rng = np.random.default_rng(11)
    n = 8
    prompts = [rng.integers(0, V - 1, size=int(rng.integers(2, 40))).tolist() for _ in range(n)]
    max_out = [int(rng.integers(4, 24)) for _ in range(n)]
    seed = 20260417
    got, acc, sub = run(desc, prompts, max_out, tau, seed, KPATS[kpat])
    exact, differs_from_greedy = check_vs_oracle(desc, prompts, max_out, got, tau, seed)
    assert exact >= n // 2, f"only {exact}/{n} requests match the oracle's sampled decode exactly"
    assert differs_from_greedy >= 2, "sampling did not change the outputs"
    if kpat != "k1":
        assert 0 < acc < sub


@pytest.mark.parametrize("exempt_rule", [1, 2])
def test_sampling_with_early_exit(exempt_rule):
    """VSD_AD_EE with sampling: the fused exit-test estimator ranks the drafted token among the
    perturbed intermediate values (the same noise the final sample uses); pruning only drops
    rows, so the committed tokens stay the target's samples (lossless vs the oracle)."""
    desc = llama.tiny(target_bigram=1.5)
    V = desc.target.vocab
    rng = np.random.default_rng(21)
    n = 8
    prompts = [rng.integers(0, V - 1, size=int(rng.integers(2, 40))).tolist() for _ in range(n)]
    max_out = [int(rng.integers(6, 24)) for _ in range(n)]
    st = {}
    # a small k_at (1 -> 4 -> 1) so the gated layers prune on this tiny pair (as in
    # tests/test_llama_gpu.py test_early_exit_decisions_given_logits)
    got, acc, sub = run(desc, prompts, max_out, 1.0, 7, KPATS["k4"], mode=abi.MODE_VSD_AD_EE,
                        gate=abi.GatePlan(1, 4, 1.0), stats=st, exit_policy=abi.ExitPolicy(1, 4, 1),
                        exempt_rule=exempt_rule)
    exact, _ = check_vs_oracle(desc, prompts, max_out, got, 1.0, 7)
    assert exact >= n // 2
    assert st.get("pruned", 0) > 0, "the estimator never pruned"


def test_sampling_drafter_invariant():
    """Same seed, different k_i patterns: the committed sequences are the same (the target's
    samples), whatever the drafter proposes."""
    desc = llama.tiny()
    V = desc.target.vocab
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, V - 1, size=int(rng.integers(2, 30))).tolist() for _ in range(6)]
    max_out = [20] * 6
    outs = [run(desc, prompts, max_out, 1.0, 99, KPATS[k])[0] for k in ("k1", "k4", "cycle")]
    same = sum(outs[0][i] == outs[1][i] == outs[2][i] for i in range(6))
    assert same >= 5, outs


def test_sampling_modes_and_arguments():
    desc = llama.tiny()
    with engine.ServingEngine(desc=desc, max_batch=2, max_seq_len=64, mode=abi.MODE_FULL,
                              default_spec_length=4, max_spec_length=8, prefill_rows=256) as eng:
        with pytest.raises(engine.FaserError):
            eng.set_sampling(1.0, 1)
        eng.set_sampling(0.0, 1)  # greedy is always allowed
    with engine.ServingEngine(desc=desc, max_batch=2, max_seq_len=64, mode=abi.MODE_VSD,
                              default_spec_length=4, max_spec_length=8, prefill_rows=256) as eng:
        with pytest.raises(engine.FaserError):
            eng.set_sampling(-1.0, 1)
        # temperature 0 after sampling: greedy again, equal to the oracle's greedy decode
        eng.set_sampling(1.0, 3)
        eng.set_sampling(0.0, 3)
        p = [5, 9, 77, 3]
        eng.submit(1, p, 12)
        while eng.live_requests():
            eng.step()
        got = eng.committed(1)
    tgt = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b)
    assert got == tgt.greedy(p, 12, desc.target.vocab - 1)
    tgt.close()


def test_sampling_config3_shapes():
    """The benchmarked shapes (config 3: 32000-entry vocabulary = 250 LM-head tiles, llama-68m
    draft / TinyLlama-1.1B target) at tau = 0.5, k = 4: outputs are the fp32 oracle's
    coupled-Gumbel samples (near-tie rule as above)."""
    desc = llama.config3()
    V = desc.target.vocab
    rng = np.random.default_rng(8)
    prompts = [rng.integers(0, V - 1, size=int(rng.integers(8, 24))).tolist() for _ in range(3)]
    max_out = [6, 5, 6]
    tau, seed = 0.5, 4242
    got, acc, sub = run(desc, prompts, max_out, tau, seed, KPATS["k4"])
    exact, _ = check_vs_oracle(desc, prompts, max_out, got, tau, seed)
    assert exact >= 1


def test_sampling_with_prefill_lane():
    """Sampling with the admission-prefill lane (the bench configuration): requests join the
    batch at different steps than without the lane, but the noise is keyed by (request,
    position) only, so the committed sequences are the oracle's samples either way."""
    desc = llama.tiny()
    V = desc.target.vocab
    rng = np.random.default_rng(17)
    n = 8
    prompts = [rng.integers(0, V - 1, size=int(rng.integers(2, 60))).tolist() for _ in range(n)]
    max_out = [int(rng.integers(4, 24)) for _ in range(n)]
    got, acc, sub = run(desc, prompts, max_out, 1.0, 555, KPATS["cycle"], prefill_lane=1)
    exact, _ = check_vs_oracle(desc, prompts, max_out, got, 1.0, 555)
    assert exact >= n // 2
    assert 0 < acc < sub

"""GPU tier: arrival-trace replay (the missing serving loop) over the Llama
path — bursty sine_segments arrivals (workload.cpp:73-114), iteration-boundary admission,
every request completes and every output is the target's greedy decode (lossless)."""
import ctypes

import numpy as np
import pytest

from oracle import lmoracle
from paper_2604_20503_b200 import abi, engine, llama, serving

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-2  # bf16 vs the fp32 oracle, relative to the row's logit range (BASELINE north star)


def test_bursty_trace_replay_lossless():
    desc = llama.tiny()
    V = desc.target.vocab
    trace = serving.synth_trace(mean_rate_per_s=400.0, peak_to_valley=10.0, duration_ms=60.0, steps=6,
                                in_range=(4, 24), out_range=(4, 20), seed=3)
    assert 5 <= len(trace) <= 60
    assert all(trace[i][0] <= trace[i + 1][0] for i in range(len(trace) - 1))
    with engine.ServingEngine(desc=desc, max_batch=6, max_seq_len=64, mode=abi.MODE_VSD,
                              default_spec_length=4, max_spec_length=8, prefill_rows=512) as eng:
        m = serving.run_trace(eng, trace, V, prompt_seed=1, fixed_k=4)
        outs = [eng.committed(j) for j in range(len(trace))]
    assert m["requests"] == len(trace) and m["completed"] == len(trace)
    assert m["tokens"] == sum(len(o) for o in outs)
    assert m["throughput_tok_s"] > 0 and m["p50_tpot_ms"] > 0 and m["p99_latency_ms"] >= m["p50_latency_ms"]
    tgt = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b, threads=2)
    try:
        for j in range(0, len(trace), max(1, len(trace) // 6)):
            prompt = engine.synth_prompt(1, j, trace[j][1], V)
            ref = tgt.greedy(prompt, trace[j][2], V - 1)
            if outs[j] != ref:  # only a near-tie of the fp32 oracle may explain a bf16 divergence
                q = next(q for q in range(min(len(outs[j]), len(ref))) if outs[j][q] != ref[q])
                z = tgt.logits(prompt + ref[:q + 1], len(prompt) + q - 1)[0][0]
                s = np.sort(z)
                assert (s[-1] - s[-2]) / (s[-1] - s[0]) <= LOGIT_TOL, (j, q)
    finally:
        tgt.close()


def test_ablation_ladder_tiny(tmp_path):
    """The four AblationModes on one trace through ModeController: every request finishes in
    every mode, outputs are identical across modes (all lossless greedy), and the summary CSV
    rows come out in the reference's order."""
    from paper_2604_20503_b200 import metrics
    desc = llama.tiny()
    V, L = desc.target.vocab, desc.target.layers
    trace = serving.synth_trace(mean_rate_per_s=300.0, peak_to_valley=4.0, duration_ms=50.0, steps=4,
                                in_range=(4, 20), out_range=(4, 16), seed=2)
    outs, sums = [], []
    for mode in (abi.MODE_VSD, abi.MODE_VSD_AD, abi.MODE_VSD_AD_EE, abi.MODE_FULL):
        with engine.ServingEngine(desc=desc, max_batch=4, max_seq_len=64, mode=mode, default_spec_length=4,
                                  max_spec_length=16, prefill_rows=512) as eng:  # AD draws k from S = {1..10}
            ctl = serving.ModeController(mode, L, fixed_k=4, gate_layer=2 if mode >= abi.MODE_VSD_AD_EE else 0,
                                         chunk=2 if mode == abi.MODE_FULL else 0)
            m = serving.run_trace(eng, trace, V, controller=ctl, num_layers=L)
            ctl.close()
            outs.append([eng.committed(j) for j in range(len(trace))])
        assert m["completed"] == len(trace) and m["summary"].finished == len(trace)
        sums.append(m["summary"])
    assert outs[1] == outs[0] and outs[2] == outs[0] and outs[3] == outs[0]
    p = tmp_path / "ablate.csv"
    metrics.write_summary_csv(p, sums)
    rows = p.read_text().splitlines()
    assert [r.split(",")[0] for r in rows[1:]] == ["VSD", "VSD_AD", "VSD_AD_EE", "FULL"]


@pytest.mark.gpu
def test_online_profiler_refreshes_during_trace():
    """The online profiler (profiler.OnlineProfiler) refits the stage-latency
    models from the engine's own per-step device timings while the trace is served, and the
    ModeController installs each refit in the AdaptiveDrafter; outputs stay the lossless ones."""
    from paper_2604_20503_b200 import profiler
    desc = llama.tiny()
    V, L = desc.target.vocab, desc.target.layers
    trace = serving.synth_trace(mean_rate_per_s=300.0, peak_to_valley=4.0, duration_ms=60.0, steps=4,
                                in_range=(4, 20), out_range=(8, 24), seed=3)
    outs = []
    for online in (False, True):
        with engine.ServingEngine(desc=desc, max_batch=4, max_seq_len=96, mode=abi.MODE_VSD_AD, default_spec_length=4,
                                  max_spec_length=16, prefill_rows=512) as eng:
            m0 = abi.LatencyModel()
            engine.lib().faser_default_latency_model(ctypes.byref(m0))
            prof = profiler.OnlineProfiler(m0, prior=[], period_steps=6, min_buckets=3) if online else None
            ctl = serving.ModeController(abi.MODE_VSD_AD, L, models=m0, profiler=prof)
            m = serving.run_trace(eng, trace, V, controller=ctl, num_layers=L)
            if online:
                prof.flush()
                assert prof.refreshes >= 1, "no refit from the runtime samples"
                assert ctl.models is not m0
                assert all(h["mape"].get("draft", 0.0) < 1.0 for h in prof.history)
            ctl.close()
            outs.append([eng.committed(j) for j in range(len(trace))])
        assert m["completed"] == len(trace)
    assert outs[1] == outs[0]

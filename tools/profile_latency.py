"""B200 stage-latency profiler + fit (replaces latmodel.cpp's synthetic
default_ground_truth for this hardware).

Measures, with the engine's own CUDA events, the draft lane (s draft steps) and the verify lane
(verify forward + accept) of config 3 for b in B_GRID, s in S_GRID (serial, steady state, no
admissions), plus the early-exit check (one gated LM-head + rank-count + compaction) and fits the
reference's load forms (latmodel.cpp:44-62) by linear least squares:
  draft   : c0*b + c1*s + c2            target : (c0*b + c1)*s + c2
  ee_check: c0*b*s + c1                 prune  : c0*b*s + c1
The share factor keeps the reference's piecewise shape, normalised to 1 at full share (serial
execution measured here). Writes profiles/r01_latency_model.json.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

B_GRID = [1, 4, 16, 32, 64, 128]
S_GRID = [1, 2, 4, 6, 8]
samples = []
REFIT = len(sys.argv) > 1 and sys.argv[1] == "--refit"
desc = llama.config3() if not REFIT else None
V = desc.target.vocab if desc else 0
rng = np.random.default_rng(0)
for b in ([] if REFIT else B_GRID):
    for mode in ("vsd", "ee"):
        eng = engine.ServingEngine(desc=desc, max_batch=b, max_seq_len=1300, default_spec_length=4,
                                   mode=abi.MODE_VSD if mode == "vsd" else abi.MODE_VSD_AD_EE,
                                   max_spec_length=16, prefill_rows=8192)
        for i in range(b):
            eng.submit(i, rng.integers(0, V - 1, size=512).tolist(), 700)
        eng.step()  # admissions + prefill
        for s in S_GRID:
            live = eng.live_requests()
            eng.set_spec_lengths(live, [s] * len(live))
            if mode == "ee":
                eng.set_gate(abi.GatePlan(11, 12, 1.0))  # one gated layer: its extra cost = T_ee
            ts = []
            for _ in range(4):
                eng.step()
                ts.append(eng.last_step_timing())
            d, v, _ = np.median(np.array(ts), axis=0)
            samples.append({"b": b, "s": s, "mode": mode, "draft_ms": float(d), "verify_ms": float(v)})
            print(json.dumps(samples[-1]), flush=True)
        eng.close()


def fit(samples):
    """The reference's load forms by least squares (the same fit the online profiler refreshes
    at run time: paper_2604_20503_b200/profiler.py fit_serial)."""
    from paper_2604_20503_b200 import profiler
    return profiler.fit_serial(samples)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--refit":
    d = json.load(open(sys.argv[2]))
    d["model"], d["mape"] = fit(d["samples"])
    json.dump(d, open(sys.argv[2], "w"), indent=1)
    print(json.dumps({"model": d["model"], "mape": d["mape"]}))
    sys.exit(0)
model, mape = fit(samples)
out = {"how": __doc__.split("\n")[0], "samples": samples, "model": model, "mape": mape}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/latency_model.json", "w"), indent=1)
print(json.dumps({"model": model, "mape": mape}))

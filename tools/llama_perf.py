"""Per-step device times of the Llama path at a given batch (VSD, fixed k)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

preset = sys.argv[1]
B = int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 4
mode = int(sys.argv[4]) if len(sys.argv) > 4 else abi.MODE_VSD
gate_layer = int(sys.argv[5]) if len(sys.argv) > 5 else 8
desc = llama.PRESETS[preset]()
V = desc.target.vocab
rng = np.random.default_rng(2)
eng = engine.ServingEngine(desc=desc, max_batch=B, max_seq_len=1400, mode=mode, default_spec_length=k,
                           max_spec_length=16, prefill_rows=8192)
for i in range(B):
    eng.submit(i, rng.integers(0, V - 1, size=int(rng.integers(128, 1024))).tolist(), 200)
eng.step()
print("prefill+first step ms", eng.last_step_timing(), flush=True)
ts = []
tok = 0
for s in range(int(os.environ.get('PERF_STEPS', 10))):
    if mode >= abi.MODE_VSD_AD_EE:
        eng.set_gate(abi.GatePlan(gate_layer, gate_layer + 1, 1.0))
    res = eng.step()
    tok += sum(r.committed for r in res)
    ts.append(eng.last_step_timing())
ts = np.array(ts)
if os.environ.get("PROFILE_ONE_STEP"):
    import torch
    torch.cuda.profiler.start()
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print(f"{preset} B={B} k={k}: draft {ts[:,0].mean():.3f} ms verify {ts[:,1].mean():.3f} ms step {ts[:,2].mean():.3f} ms; "
      f"{tok / (ts[:,2].sum() / 1e3):.0f} tok/s device; launches {eng.kernel_launches()}")

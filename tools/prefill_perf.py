"""Device time of single-prompt admissions (prefill of one prompt + one 1-token round), the
unit of work continuous batching adds per admitted request. Usage: prefill_perf.py preset len n"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

preset, plen, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
desc = llama.PRESETS[preset]()
V = desc.target.vocab
rng = np.random.default_rng(1)
with engine.ServingEngine(desc=desc, max_batch=8, max_seq_len=plen + 16, mode=abi.MODE_VSD, default_spec_length=1,
                          max_spec_length=4, prefill_rows=8192) as eng:
    ts = []
    for i in range(n + 2):
        eng.submit(i, rng.integers(0, V - 1, size=plen).tolist(), 1)
        eng.step()
        ts.append(eng.last_step_timing())
    t = np.array(ts[2:])
    print(f"{preset} prompt {plen}: admission step {t[:, 2].mean():.3f} ms (draft+prefill {t[:, 0].mean():.3f}, "
          f"verify {t[:, 1].mean():.3f})")

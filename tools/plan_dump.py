"""Print the GEMM launch plan (bn, splits, mc) the planner picks for the config-3/4 shapes."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import engine  # noqa: E402
L = engine.lib()
for name, (n, k) in {"qkv": (2560, 2048), "o": (2048, 2048), "gu": (11264, 2048), "down": (2048, 5632),
                     "lm": (32000, 2048), "d_qkv": (2304, 768), "d_o": (768, 768), "d_gu": (6144, 768),
                     "d_down": (768, 3072), "d_lm": (32000, 768)}.items():
    for t in (4, 32, 128, 256, 512):
        out = (C.c_int32 * 4)()
        L.faser_k_gemm_plan(n, t, k, out)
        print(name, t, list(out))

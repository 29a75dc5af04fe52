"""GPU tier: the persistent single-launch forward (mega.cu, opt-in FASER_MEGA=1) on the Llama
path — every finished request must equal the fp32 oracle's greedy decode (a divergence only
where the oracle's top-2 gap is inside the bf16 tolerance), like the per-layer-launch path."""
import os

import numpy as np
import pytest

from oracle import lmoracle
from paper_2604_20503_b200 import abi, engine, llama

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-2


@pytest.mark.parametrize("preset", ["tiny", "tp_tiny"])
def test_persistent_forward_lossless(preset, monkeypatch):
    monkeypatch.setenv("FASER_MEGA", "1")
    desc = llama.PRESETS[preset]()
    V = desc.target.vocab
    rng = np.random.default_rng(11)
    prompts = [rng.integers(0, V - 1, size=int(rng.integers(3, 50))).tolist() for _ in range(9)]
    max_out = [int(rng.integers(2, 30)) for _ in range(9)]
    with engine.ServingEngine(desc=desc, max_batch=5, max_seq_len=128, mode=abi.MODE_VSD, default_spec_length=4,
                              max_spec_length=8, prefill_rows=1024) as eng:
        for i, (p, m) in enumerate(zip(prompts, max_out)):
            eng.submit(i, p, m)
        ks = [1, 3, 4, 6, 8]
        s = 0
        while eng.live_requests():
            live = eng.live_requests()
            eng.set_spec_lengths(live, [ks[(r + s) % len(ks)] for r in live])
            eng.step()
            s += 1
        got = [eng.committed(i) for i in range(len(prompts))]
    tgt = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b, threads=2)
    try:
        for i, (p, m) in enumerate(zip(prompts, max_out)):
            want = tgt.greedy(p, m, V - 1)
            if got[i] != want:
                q = next(q for q in range(min(len(got[i]), len(want))) if got[i][q] != want[q])
                z = tgt.logits(p + want[:q + 1], len(p) + q - 1)[0][0]
                srt = np.sort(z)
                assert (srt[-1] - srt[-2]) / (srt[-1] - srt[0]) <= LOGIT_TOL, (i, q)
    finally:
        tgt.close()

"""Generate tests/golden/toy_golden.json from the REFERENCE itself (oracle/_ref, the
reference's own toylm/sdcore/exitctl/workload TUs compiled in place from /root/reference).

Run here (the reference is not on the GPU box):  python tests/golden/make_golden.py
The JSON is committed; tests compare the restated oracle and the CUDA engine against it.
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402
from paper_2604_20503_b200 import abi  # noqa: E402


def digest(records):
    h = hashlib.sha256()
    for r in records:
        h.update(repr(r).encode())
    return h.hexdigest()


def episode(ref, p, n, max_batch, early_exit, k_mode, fixed_k=4, k_seed=7, in_range=(4, 12),
            out_range=(16, 48)):
    inl, outl = po.backlog_lengths(1, n, in_range, out_range)
    prompts = [ref.synth_prompt(1, i, inl[i], p.vocab) for i in range(n)]
    cfg = abi.EpisodeCfg(model=p, max_batch=max_batch, early_exit=early_exit, k_mode=k_mode,
                         fixed_k=fixed_k, exempt_rule=1, threads=1, k_seed=k_seed,
                         policy=abi.ExitPolicy.default(), gate=abi.GatePlan(8, 32, 1.0))
    outs, log, st = ref.run_episode(cfg, prompts, outl, log_cap=200000)
    recs = [r.as_tuple() for r in log]
    return {
        "n": n, "max_batch": max_batch, "early_exit": early_exit, "k_mode": k_mode,
        "fixed_k": fixed_k, "k_seed": k_seed, "divergence": p.divergence,
        "in_len": inl, "out_len": outl, "outputs": outs,
        "stats": {k: getattr(st, k) for k in ("rounds", "drafted", "submitted", "accepted",
                                                 "committed", "false_prunes", "finished",
                                                 "layer_work", "layer_work_full")},
        "n_records": len(recs), "records_sha256": digest(recs),
        "first_records": [list(map(lambda x: list(x) if isinstance(x, tuple) else x, r))
                          for r in recs[:40]],
    }


def main():
    ref = po.ref()
    p = abi.ToyParams.default()
    g = {"source": "oracle/_ref/libspecsim_ref.so (reference TUs compiled in place)",
         "params": {"seed": 1, "vocab": 64, "layers": 32, "order": 2, "divergence": 0.3,
                    "noise_seed": 2, "logit_scale": 4.0, "noise_scale": 1.0}}
    prompts = [ref.synth_prompt(1, i, 8, 64) for i in range(16)]
    g["synth_prompt_seed1_len8"] = prompts
    g["ar_decode_24"] = [ref.autoregressive_decode(p, pr, 24) for pr in prompts]
    zf, zn = ref.final_and_noise(p, prompts[:4])
    g["z_final_rows0_3"] = [[float.hex(float(x)) for x in row] for row in zf]
    g["z_noise_rows0_3"] = [[float.hex(float(x)) for x in row] for row in zn]
    lay = [1, 8, 16, 31, 32]
    g["target_logits_row0"] = {str(l): [float.hex(float(x)) for x in ref.target_logits(p, [prompts[0]], [l])[0]]
                               for l in lay}
    pol = abi.ExitPolicy.default()
    g["k_at_L32"] = [ref.k_at(pol, l, 32) for l in range(0, 33)]
    # draft/target single-step agreement vs eta over 2000 seeded prefixes
    pre = [ref.synth_prompt(5, i, 1 + i % 24, 64) for i in range(2000)]
    agree = {}
    for eta in (0.0, 0.25, 0.3, 0.5, 0.75, 1.0):
        q = abi.ToyParams.default(divergence=eta)
        t = ref.target_next(q, pre)
        d = ref.draft_next(q, pre)
        agree[str(eta)] = float((t == d).mean())
    g["agreement_vs_eta_2000"] = agree
    g["episodes"] = {
        "cfg1_vsd_b4_k4": episode(ref, p, 4, 4, 0, 0),
        "cfg1_ee_b4_k4": episode(ref, p, 4, 4, 1, 0),
        "cfg2_ee_b32_dyn": episode(ref, p, 32, 32, 1, 1),
        "cfg2_ee_b32_dyn_eta05": episode(ref, abi.ToyParams.default(divergence=0.5), 32, 32, 1, 1),
        "b256_vsd_k4_backlog300": episode(ref, p, 300, 256, 0, 0),
    }
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "toy_golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()

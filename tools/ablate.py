"""Ablation ladder on B200 (the reference's `ablate` command): the SAME bursty
arrival trace and seed served by VSD, VSD_AD, VSD_AD_EE and FULL on the same kernels; writes the
reference's wire formats — one metrics JSON-lines file per mode and a 4-row summary CSV
(metrics.cpp:68-113) — and prints the table.

  python tools/ablate.py [--workload cfg3] [--seconds 10] [--rate 60] [--batch 64] [--k 4]
                         [--gate-layer 0] [--chunk 0] --out profiles/r01_ablation_cfg3
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama, metrics, serving  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--seconds", type=float, default=10.0)
    ap.add_argument("--rate", type=float, default=60.0)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--gate-layer", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--in-range", default="128,1024")
    ap.add_argument("--out-range", default="64,256")
    ap.add_argument("--out", default="gpurun_out/ablation")
    ap.add_argument("--modes", default="VSD,VSD_AD,VSD_AD_EE,FULL")
    ap.add_argument("--refresh-steps", type=int, default=0,
                    help="online profiler: refit the latency models from runtime samples every N steps (0 = off)")
    args = ap.parse_args()
    desc = llama.PRESETS[args.workload]()
    V, L = desc.target.vocab, desc.target.layers
    in_r = tuple(int(v) for v in args.in_range.split(","))
    out_r = tuple(int(v) for v in args.out_range.split(","))
    trace = serving.synth_trace(mean_rate_per_s=args.rate, peak_to_valley=10.0, duration_ms=args.seconds * 1e3,
                                steps=12, in_range=in_r, out_range=out_r, seed=1)
    models = llama.fitted_latency_model() if args.workload != "tiny" else None
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    summaries = []
    names = {"VSD": abi.MODE_VSD, "VSD_AD": abi.MODE_VSD_AD, "VSD_AD_EE": abi.MODE_VSD_AD_EE, "FULL": abi.MODE_FULL}
    for mode in [names[m] for m in args.modes.split(",")]:
        with engine.ServingEngine(desc=desc, max_batch=args.batch, max_seq_len=in_r[1] + out_r[1] + 8, mode=mode,
                                  default_spec_length=args.k, max_spec_length=16, prefill_rows=8192) as eng:
            for i in range(min(4, args.batch)):  # warm-up requests outside the trace
                eng.submit(10 ** 9 + i, [1 + i, 2, 3, 4, 5], 8)
            while eng.pending_work() > 0:
                eng.step()
            prof = None
            if args.refresh_steps and models is not None:
                from paper_2604_20503_b200 import profiler
                # the offline grid is config 3's (tools/profile_latency.py): a prior only for it
                prior = profiler.offline_samples() if args.workload == "cfg3" else None
                prof = profiler.OnlineProfiler(models, prior=prior, period_steps=args.refresh_steps)
            ctl = serving.ModeController(mode, L, fixed_k=args.k, models=models, gate_layer=args.gate_layer,
                                         chunk=args.chunk, profiler=prof)
            m = serving.run_trace(eng, trace, V, prompt_seed=1, controller=ctl, num_layers=L, seed=1)
            if prof is not None:
                smp, n_rt = prof.samples()
                print(json.dumps({"mode": mode, "online_refits": prof.refreshes, "history": prof.history[-3:],
                                  "runtime_buckets": n_rt, "samples": smp[-n_rt:][:40],
                                  "model": profiler.model_dict(ctl.models)}), flush=True)
            ctl.close()
        s = m["summary"]
        summaries.append(s)
        metrics.write_metrics_jsonl(f"{args.out}_{s.mode}.jsonl", s)
        print(json.dumps({"mode": s.mode, "throughput_tok_s": round(s.throughput_tok_s, 1),
                          "p50_tpot_ms": round(m["p50_tpot_ms"], 3), "mean_tpot_ms": round(s.mean_tpot_ms, 3),
                          "p50_latency_ms": round(s.p50_request_latency_ms, 1),
                          "acceptance": round(s.acceptance_ratio, 3),
                          "layer_work_frac": round(s.layer_work / max(s.layer_work_full, 1), 3),
                          "overlap_iterations": s.overlap_iterations, "iterations": s.iterations}), flush=True)
    metrics.write_summary_csv(f"{args.out}.csv", summaries)
    print(open(f"{args.out}.csv").read())


if __name__ == "__main__":
    main()

"""Lane profiler: the SM-share dimension of the stage latency models, measured on B200 green-context
partitions, plus the co-run interference of the overlapped lanes (PAPER.md:541-568,
575; latmodel.hpp:10-31 model form; overlap.hpp:11-65).

For config 3 at b in B_GRID, s in S_GRID (steady state, all requests resident):
  serial      : draft + verify on the whole GPU (r = 1)                -> draft(b,s,1), target(b,s,1)
  partitioned : one chunk, the draft on round8(r*SMs) SMs, then the verify on the rest
                (overlap chunk = s, r in R_GRID)                       -> draft(b,s,r), target(b,s,1-r)
  overlapped  : chunk = s/2 at r, lanes co-running, and the same partitions/chunks serialised
                (lane_mode isolated): per-chunk co-run / isolated time = interference
Fit (restating latmodel.cpp's model form, not its ALS code): load terms by least squares on the
serial samples (draft c0*b + c1*s + c2, target (c0*b + c1)*s + c2), then the share factor
factor(x) = a1 - g1*x (x <= knee), a2 - g2*x (x > knee), continuous at the knee, by exhaustive
knee search over the measured shares + least squares, normalised to factor(knee) = 1 (the load
term absorbs the scale, as fit_stage does). Writes gpurun_out/lane_profile.json.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402

B_GRID = [int(x) for x in os.environ.get("LP_B", "8,32,64,128").split(",")]
S_GRID = [int(x) for x in os.environ.get("LP_S", "2,4,6").split(",")]
R_GRID = [float(x) for x in os.environ.get("LP_R", "0.25,0.5,0.75").split(",")]
REPS = 3


def med_step(eng, live, s, overlap):
    eng.set_spec_lengths(live, [s] * len(live))
    d, v, tl = [], [], []
    for _ in range(REPS):
        if overlap is None:
            eng.set_overlap(False)
        else:
            eng.set_overlap(True, *overlap)
        eng.step()
        t = eng.last_step_timing()
        d.append(t[0])
        v.append(t[2])
        if overlap is not None:
            tl.append(eng.last_timeline())
    return float(np.median(d)), float(np.median(v)), tl


def chunk_times(tl, kind):
    out = {}
    for info, evs in tl:
        for e in evs:
            if e.kind == kind:
                out.setdefault(e.chunk, []).append(e.end_ms - e.start_ms)
    return {q: float(np.median(x)) for q, x in out.items()}


def main():
    desc = llama.config3()
    V = desc.target.vocab
    rng = np.random.default_rng(0)
    samples, interference, step_cmp = [], [], []
    for b in B_GRID:
        eng = engine.ServingEngine(desc=desc, max_batch=b, max_seq_len=1800, default_spec_length=4,
                                   mode=abi.MODE_FULL, max_spec_length=16, prefill_rows=8192)
        for i in range(b):
            eng.submit(i, rng.integers(0, V - 1, size=512).tolist(), 1200)
        eng.set_overlap(False)
        eng.step()  # admissions + prefill
        live = eng.live_requests()
        for s in S_GRID:
            med_step(eng, live, s, None)  # warm the shapes
            full_d, full_st, _ = med_step(eng, live, s, None)
            t_ser = full_st - full_d  # verify + accept on the whole GPU
            samples.append({"stage": "draft", "b": b, "s": s, "r": 1.0, "ms": full_d})
            samples.append({"stage": "target", "b": b, "s": s, "r": 0.0, "ms": t_ser})
            for r in R_GRID:
                _, _, tl = med_step(eng, live, s, (s, r))
                dr = chunk_times(tl, abi.EV_DRAFT_CHUNK).get(0)
                vr = chunk_times(tl, abi.EV_VERIFY_CHUNK).get(0)
                info = tl[-1][0]
                samples.append({"stage": "draft", "b": b, "s": s, "r": r, "ms": dr, "sms": info.draft_sms})
                samples.append({"stage": "target", "b": b, "s": s, "r": r, "ms": vr, "sms": info.verify_sms})
                if s >= 4:
                    c = s // 2
                    eng.set_lane_mode(abi.LANES_OVERLAP)
                    _, st_ov, tl_ov = med_step(eng, live, s, (c, r))
                    eng.set_lane_mode(abi.LANES_ISOLATED)
                    _, st_iso, tl_iso = med_step(eng, live, s, (c, r))
                    eng.set_lane_mode(abi.LANES_OVERLAP)
                    dco, diso = chunk_times(tl_ov, abi.EV_DRAFT_CHUNK), chunk_times(tl_iso, abi.EV_DRAFT_CHUNK)
                    vco, viso = chunk_times(tl_ov, abi.EV_VERIFY_CHUNK), chunk_times(tl_iso, abi.EV_VERIFY_CHUNK)
                    rec = {"b": b, "s": s, "chunk": c, "r": r, "draft_sms": info.draft_sms,
                           "verify_sms": info.verify_sms, "step_ms_overlapped": st_ov, "step_ms_isolated": st_iso,
                           "step_ms_serial_whole_gpu": full_st,
                           "draft_chunk_ms": {"corun": dco, "isolated": diso},
                           "verify_chunk_ms": {"corun": vco, "isolated": viso},
                           "interference_verify": {q: vco[q] / viso[q] for q in vco if q in viso and viso[q] > 0},
                           "interference_draft": {q: dco[q] / diso[q] for q in dco if q in diso and diso[q] > 0}}
                    interference.append(rec)
                    print(json.dumps(rec), flush=True)
            print(json.dumps([x for x in samples if x["b"] == b and x["s"] == s]), flush=True)
        eng.close()
    model, mape = fit(samples)
    out = {"how": __doc__.split("\n")[0], "samples": samples, "model": model, "mape": mape,
           "interference": interference}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/lane_profile.json", "w"), indent=1)
    print(json.dumps({"model": model, "mape": mape}))


def fit(samples):
    def lstsq(rows, y):
        c, *_ = np.linalg.lstsq(np.array(rows, float), np.array(y, float), rcond=None)
        return c

    dr = [x for x in samples if x["stage"] == "draft" and x["ms"]]
    tg = [x for x in samples if x["stage"] == "target" and x["ms"]]
    ser_d = [x for x in dr if x["r"] == 1.0]
    ser_t = [x for x in tg if x["r"] == 0.0]
    cd = lstsq([[x["b"], x["s"], 1.0] for x in ser_d], [x["ms"] for x in ser_d])
    if cd[2] < 0:  # every prediction must stay positive (eval_latency > 0): no intercept then
        c2 = lstsq([[x["b"], x["s"]] for x in ser_d], [x["ms"] for x in ser_d])
        cd = np.array([c2[0], c2[1], 0.0])
    ct = lstsq([[x["b"] * x["s"], x["s"], 1.0] for x in ser_t], [x["ms"] for x in ser_t])
    if ct[2] < 0:
        c2 = lstsq([[x["b"] * x["s"], x["s"]] for x in ser_t], [x["ms"] for x in ser_t])
        ct = np.array([c2[0], c2[1], 0.0])
    load = {"draft": lambda x: cd[0] * x["b"] + cd[1] * x["s"] + cd[2],
            "target": lambda x: (ct[0] * x["b"] + ct[1]) * x["s"] + ct[2]}
    own = {"draft": lambda x: x["r"], "target": lambda x: 1.0 - x["r"]}
    model, mape = {}, {}
    for stage, xs, c in (("draft", dr, cd), ("target", tg, ct)):
        pts = [(own[stage](x), x["ms"] / load[stage](x), x) for x in xs]
        best = None
        for knee in sorted({p[0] for p in pts if p[0] < 1.0}):
            # f = a1 - g1 x (x <= K); f = a1 - g1 K - g2 (x - K) (x > K): linear in (a1, g1, g2)
            A = [[1.0, -x if x <= knee else -knee, 0.0 if x <= knee else -(x - knee)] for x, _, _ in pts]
            y = [f for _, f, _ in pts]
            a1, g1, g2 = lstsq(A, y)
            err = float(np.sum((np.array(A) @ np.array([a1, g1, g2]) - np.array(y)) ** 2))
            if best is None or err < best[0]:
                best = (err, knee, a1, g1, g2)
        _, knee, a1, g1, g2 = best
        a2 = a1 - g1 * knee + g2 * knee
        fk = a1 - g1 * knee  # normalise: factor(knee) = 1, the load absorbs the scale
        p = {"stage": {"draft": 0, "target": 1}[stage], "knee": knee, "a1": a1 / fk, "gamma1": g1 / fk,
             "a2": a2 / fk, "gamma2": g2 / fk, "c0": c[0] * fk, "c1": c[1] * fk, "c2": c[2] * fk}
        model[stage] = {k: float(v) for k, v in p.items()}

        def pred(x, p=p, stage=stage):
            xo = own[stage](x)
            f = p["a1"] - p["gamma1"] * xo if xo <= p["knee"] else p["a2"] - p["gamma2"] * xo
            ld = p["c0"] * x["b"] + p["c1"] * x["s"] + p["c2"] if stage == "draft" else \
                (p["c0"] * x["b"] + p["c1"]) * x["s"] + p["c2"]
            return f * ld
        mape[stage] = float(np.mean([abs(pred(x) - x["ms"]) / x["ms"] for x in xs]))
    return model, mape


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--refit":
        d = json.load(open(sys.argv[2]))
        d["model"], d["mape"] = fit(d["samples"])
        json.dump(d, open(sys.argv[2], "w"), indent=1)
        print(json.dumps({"model": d["model"], "mape": d["mape"]}))
    else:
        main()

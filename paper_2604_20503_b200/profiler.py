"""Online stage-latency profiler: the serving loop's runtime samples refit the latency models the
controllers plan with.

Reference behaviour: FASER fits draft / target / early-exit latency models offline and
"refreshes the profilers every 2 hours in a separate process using runtime execution statistics"
(the load forms are latmodel.cpp:44-62, the share factor latmodel.cpp:32-43).
Here:

* ``fit_serial(samples)`` is the least-squares fit of the reference's load forms over serial
  (whole-GPU) stage samples — the fit tools/profile_latency.py applies to its offline b x s grid:
    draft    : c0*b + c1*s + c2          target : (c0*b + c1)*s + c2
    ee_check : c0*b*s + c1               prune  : 0.1 x ee_check
  Each sample is divided by the model's share factor at the serial share (own share 1), so the
  fitted load composes with the SM-share factor of tools/lane_profile.py unchanged.
* ``OnlineProfiler`` collects one sample per executed serial step from the running engine (b,
  the draft loop's length max k_i, the verify's mean length, device-event stage times), keeps a
  bounded window per (b, s) bucket, and every ``period_steps`` steps (or ``period_s`` seconds)
  refits on a background worker thread, off the serving loop. Runtime buckets replace the
  offline profile's sample of the same (b, s); buckets the serving load never visits keep their
  offline sample, so the fit stays determined when the runtime batch sizes are narrow. A
  finished refit is picked up by ``poll()``; ``serving.ModeController`` installs it in the
  AdaptiveDrafter (faser_drafter_set_models) and in its gate / overlap planning.
"""
import json
import os
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import abi

STAGES = ("draft", "target", "ee_check", "prune")
PROFILE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "r01_latency_model.json")


def serial_factor(p):
    """latmodel.cpp:32-43 share factor at own share x = 1 (whole GPU): a2 - gamma2 * 1, or the
    first segment when the knee is at 1."""
    p = p if isinstance(p, dict) else params_dict(p)
    return p["a1"] - p["gamma1"] if p["knee"] >= 1.0 else p["a2"] - p["gamma2"]


def params_dict(p):
    return {n: float(getattr(p, n)) for n, _ in abi.LatencyParams._fields_ if n != "reserved0"}


def model_dict(m):
    return {s: params_dict(getattr(m, s)) for s in STAGES}


def to_model(d):
    out = abi.LatencyModel()
    for name in STAGES:
        p = getattr(out, name)
        for k, v in d[name].items():
            setattr(p, k, int(v) if k == "stage" else float(v))
    return out


def _lstsq(rows, y):
    """Least squares in relative error (each row weighted by 1/y: stage times span 0.1-10 ms, and
    the planners compare ratios); None when the design is rank-deficient (e.g. a serving load
    that only ever ran one speculative length: the stage keeps its previous coefficients)."""
    A = np.array(rows, float)
    if np.linalg.matrix_rank(A) < A.shape[1]:
        return None
    y = np.array(y, float)
    w = 1.0 / np.maximum(np.abs(y), 1e-6)
    c, *_ = np.linalg.lstsq(A * w[:, None], y * w, rcond=None)
    return c


def fit_serial(samples, base=None):
    """Least-squares loads over serial samples {b, s, mode ('vsd' | 'ee'), draft_ms, verify_ms
    [, s_verify, ee_layers]}: returns (model dict, mape dict). ``base`` (model dict) supplies the
    share-factor shape of each stage and the fallback for a stage with too few samples; without
    it the reference's default shape (knee 0.5) with factor 1 at the serial share is used."""
    shape = {"knee": 0.5, "a1": 1.575, "gamma1": 0.9, "a2": 1.25, "gamma2": 0.25}
    base = base or {s: {"stage": float(i), **shape, "c0": 0.0, "c1": 0.0, "c2": 0.0}
                    for i, s in enumerate(STAGES)}
    out = {s: dict(base[s]) for s in STAGES}
    fd, ft, fe = (serial_factor(base[s]) for s in ("draft", "target", "ee_check"))
    vs = [x for x in samples if x.get("mode", "vsd") == "vsd"]
    sv = lambda x: x.get("s_verify", x["s"])  # noqa: E731
    mape = {}
    cd = ct = ce = None
    dr = [x for x in samples if x.get("draft_ms", 0) > 0]
    if len({(x["b"], x["s"]) for x in dr}) >= 3:
        cd = _lstsq([[x["b"], x["s"], 1.0] for x in dr], [x["draft_ms"] / fd for x in dr])
    if cd is not None:
        if cd[2] < 0:  # keep every prediction positive (eval_latency > 0): refit without intercept
            c2 = _lstsq([[x["b"], x["s"]] for x in dr], [x["draft_ms"] / fd for x in dr])
            cd = np.array([c2[0], c2[1], 0.0]) if c2 is not None else None
    if cd is not None:
        out["draft"].update(c0=float(cd[0]), c1=float(cd[1]), c2=float(cd[2]))
        pd = lambda x: fd * (cd[0] * x["b"] + cd[1] * x["s"] + cd[2])  # noqa: E731
        mape["draft"] = float(np.mean([abs(pd(x) - x["draft_ms"]) / x["draft_ms"] for x in dr]))
    if len({(x["b"], sv(x)) for x in vs}) >= 3:
        ct = _lstsq([[x["b"] * sv(x), sv(x), 1.0] for x in vs], [x["verify_ms"] / ft for x in vs])
    if ct is not None:
        out["target"].update(c0=float(ct[0]), c1=float(ct[1]), c2=float(ct[2]))
        pt = lambda x: ft * ((ct[0] * x["b"] + ct[1]) * sv(x) + ct[2])  # noqa: E731
        mape["target"] = float(np.mean([abs(pt(x) - x["verify_ms"]) / x["verify_ms"] for x in vs]))
    # ee_check: the verify time an EE step pays above the target model, per gated layer
    tp = out["target"]
    ee = []
    for x in samples:
        if x.get("mode") == "ee":
            tgt = ft * ((tp["c0"] * x["b"] + tp["c1"]) * sv(x) + tp["c2"])
            ee.append((x["b"], sv(x), (x["verify_ms"] - tgt) / max(x.get("ee_layers", 1), 1)))
    if len({(b, s) for b, s, _ in ee}) >= 2:
        ce = _lstsq([[b * s, 1.0] for b, s, _ in ee], [max(d, 1e-3) / fe for _, _, d in ee])
    if ce is not None:
        ce = np.maximum(ce, [0.0, 1e-3])
        out["ee_check"].update(c0=float(ce[0]), c1=float(ce[1]), c2=0.0)
        # row compaction is folded into the measured ee_check delta; pruning itself ~10 % of it
        out["prune"].update(c0=float(ce[0]) * 0.1, c1=float(ce[1]) * 0.1, c2=0.0)
    return out, mape


def offline_samples(path=PROFILE):
    try:
        with open(path) as f:
            return list(json.load(f)["samples"])
    except (OSError, KeyError, ValueError):
        return []


class OnlineProfiler:
    """Runtime samples -> periodic background refit -> refreshed abi.LatencyModel.

    record() is called once per executed step by the serving loop; only serial steps (draft SM
    share r = 1, no overlap) are samples of the whole-GPU loads. ``window`` bounds the samples
    kept per (b, s) bucket (the newest win); a bucket's sample is its median."""

    def __init__(self, base_model, prior=None, period_steps=256, period_s=0.0, window=16, min_buckets=3):
        """``prior``: the offline grid of the SAME model pair (e.g. offline_samples() for config
        3, whose grid profiles/r01_latency_model.json holds); None = runtime samples only."""
        self.base = model_dict(base_model) if not isinstance(base_model, dict) else base_model
        self.prior = list(prior) if prior is not None else []
        self.period_steps, self.period_s, self.window, self.min_buckets = period_steps, period_s, window, min_buckets
        self.buckets = {}
        self.lock = threading.Lock()
        self.pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="faser-profiler")
        self.future = None
        self.steps_since = 0
        self.t_last = time.monotonic()
        self.refreshes = 0
        self.history = []  # (step count at submit, mape) per installed refit
        self.steps = 0

    def record(self, b, ks, draft_ms, verify_ms, r=1.0, ee_layers=0):
        """One executed step: b live requests drafting ks (list of k_i), device stage times."""
        self.steps += 1
        self.steps_since += 1
        if b <= 0 or not ks or r < 1.0 or verify_ms <= 0:
            return
        s = int(max(ks))
        key = (int(b), s, "ee" if ee_layers else "vsd")
        x = {"b": int(b), "s": s, "s_verify": float(np.mean(ks)), "mode": key[2], "draft_ms": float(draft_ms),
             "verify_ms": float(verify_ms), "ee_layers": int(ee_layers)}
        with self.lock:
            q = self.buckets.setdefault(key, [])
            q.append(x)
            del q[:-self.window]

    def samples(self):
        """Runtime bucket medians, plus the offline samples of buckets not seen at runtime."""
        with self.lock:
            rt = {}
            for key, q in self.buckets.items():
                m = {"b": key[0], "s": key[1], "mode": key[2], "ee_layers": q[-1]["ee_layers"]}
                for f in ("s_verify", "draft_ms", "verify_ms"):
                    m[f] = float(np.median([x[f] for x in q]))
                rt[key] = m
        seen = set(rt)
        out = [dict(x) for x in self.prior if (x["b"], x["s"], x.get("mode", "vsd")) not in seen]
        return out + list(rt.values()), len(rt)

    def due(self):
        if self.future is not None:
            return False
        if self.period_s > 0 and time.monotonic() - self.t_last >= self.period_s:
            return True
        return self.period_steps > 0 and self.steps_since >= self.period_steps

    def poll(self):
        """Submits a refit when one is due and returns a finished one (abi.LatencyModel) once."""
        got = None
        if self.future is not None and self.future.done():
            res = self.future.result()
            self.future = None
            if res is not None:
                model, mape = res
                self.base = model
                self.refreshes += 1
                self.history.append({"step": self.steps, "mape": mape})
                got = to_model(model)
        if self.due():
            smp, n_rt = self.samples()
            self.steps_since = 0
            self.t_last = time.monotonic()
            if n_rt >= 1 and len({(x["b"], x["s"]) for x in smp}) >= self.min_buckets:
                self.future = self.pool.submit(fit_serial, smp, self.base)
        return got

    def flush(self):
        """Waits for a refit in flight (tests / end of a run) and returns it like poll()."""
        if self.future is not None:
            self.future.result()
        return self.poll() if self.future is not None else None

    def close(self):
        self.pool.shutdown(wait=True)

"""CPU tier: the online latency profiler (profiler.py): the least-squares
refit of the reference's load forms (latmodel.cpp:44-62), the periodic background refresh from
runtime samples, and its installation into the AdaptiveDrafter through the C ABI
(faser_drafter_set_models) and the ModeController's planning models."""
import ctypes as C

import numpy as np
import pytest

from paper_2604_20503_b200 import abi, controller, engine, profiler, serving

TRUE = {"draft": (0.004, 0.13, 0.05), "target": (0.006, 0.01, 1.2), "ee_check": (2e-4, 0.04)}


def base_model():
    m = engine.default_latency_model() if hasattr(engine, "default_latency_model") else None
    d = {s: {"stage": float(i), "knee": 0.5, "a1": 2.0, "gamma1": 2.0, "a2": 1.2, "gamma2": 0.4,
             "c0": 0.0, "c1": 0.0, "c2": 0.0} for i, s in enumerate(profiler.STAGES)}
    return m, d


def synth(b, s, factor=0.8, ee_layers=0):
    cd, ct, ce = TRUE["draft"], TRUE["target"], TRUE["ee_check"]
    draft = factor * (cd[0] * b + cd[1] * s + cd[2])
    verify = factor * ((ct[0] * b + ct[1]) * s + ct[2])
    if ee_layers:
        verify += ee_layers * factor * (ce[0] * b * s + ce[1])
    return draft, verify


def test_fit_serial_recovers_load_forms():
    _, base = base_model()
    f = profiler.serial_factor(base["draft"])
    assert f == pytest.approx(0.8)
    smp = []
    for b in (1, 8, 32, 128):
        for s in (1, 2, 4, 6):
            d, v = synth(b, s, f)
            smp.append({"b": b, "s": s, "mode": "vsd", "draft_ms": d, "verify_ms": v})
            d, v = synth(b, s, f, ee_layers=2)
            smp.append({"b": b, "s": s, "mode": "ee", "draft_ms": d, "verify_ms": v, "ee_layers": 2})
    m, mape = profiler.fit_serial(smp, base)
    assert [m["draft"][k] for k in ("c0", "c1", "c2")] == pytest.approx(TRUE["draft"], rel=1e-6, abs=1e-9)
    assert [m["target"][k] for k in ("c0", "c1", "c2")] == pytest.approx(TRUE["target"], rel=1e-6, abs=1e-9)
    assert [m["ee_check"][k] for k in ("c0", "c1")] == pytest.approx(TRUE["ee_check"], rel=1e-6, abs=1e-9)
    assert mape["draft"] < 1e-9 and mape["target"] < 1e-9
    # share-factor shape kept from the base model
    assert m["target"]["a1"] == base["target"]["a1"] and m["draft"]["knee"] == base["draft"]["knee"]
    # the refit evaluates through the native eval_latency exactly like the generating forms
    lm = profiler.to_model(m)
    out = C.c_double()
    engine._check(engine.lib().faser_eval_latency(C.byref(lm), 1, C.c_double(32), C.c_double(4),
                                                  C.c_double(0.0), C.byref(out)))
    assert out.value == pytest.approx(synth(32, 4, f)[1], rel=1e-9)


def test_online_refresh_from_runtime_samples():
    _, base = base_model()
    f = profiler.serial_factor(base["draft"])
    # prior (offline grid) from a different "hardware": every load 2x
    prior = []
    for b in (1, 4, 16, 64):
        for s in (1, 4, 8):
            d, v = synth(b, s, f)
            prior.append({"b": b, "s": s, "mode": "vsd", "draft_ms": 2 * d, "verify_ms": 2 * v})
    prof = profiler.OnlineProfiler(base, prior=prior, period_steps=20, window=8)
    rng = np.random.default_rng(0)
    got = []
    for step in range(200):
        b = int(rng.choice([1, 4, 16, 64]))
        ks = [int(rng.choice([1, 4, 8]))] * b
        d, v = synth(b, max(ks), f)
        prof.record(b, ks, d, v)
        m = prof.poll()
        if m is not None:
            got.append(m)
        if step == 3:
            assert prof.future is None  # not due before period_steps
        if prof.future is not None:  # let the background refit finish (deterministic count)
            prof.future.result()
    m = prof.flush() or (got[-1] if got else None)
    assert prof.refreshes >= 3 and m is not None
    # every runtime bucket replaced its 2x prior sample: the refit is the runtime model
    assert m.target.c2 == pytest.approx(TRUE["target"][2], rel=1e-6)
    assert m.draft.c1 == pytest.approx(TRUE["draft"][1], rel=1e-6)
    # overlapped (r < 1) steps are not serial samples
    n = sum(len(q) for q in prof.buckets.values())
    prof.record(8, [4] * 8, 9.0, 9.0, r=0.5)
    assert sum(len(q) for q in prof.buckets.values()) == n
    prof.close()


def test_unseen_buckets_keep_offline_samples():
    _, base = base_model()
    prior = [{"b": b, "s": s, "mode": "vsd", "draft_ms": 1.0 + b, "verify_ms": 2.0 + s} for b in (1, 2) for s in (1, 2)]
    prof = profiler.OnlineProfiler(base, prior=prior, period_steps=1)
    prof.record(2, [2, 2], 5.0, 7.0)
    smp, n_rt = prof.samples()
    assert n_rt == 1 and len(smp) == 4
    assert {"b": 2, "s": 2} == {k: v for k, v in smp[-1].items() if k in ("b", "s")}
    assert smp[-1]["draft_ms"] == 5.0
    prof.close()


def test_drafter_set_models_and_controller_install():
    _, base = base_model()
    m0 = profiler.to_model(base)
    d = controller.AdaptiveDrafter(models=m0)
    d.set_models(profiler.to_model(base))
    with pytest.raises(engine.FaserError):
        engine._check(engine.lib().faser_drafter_set_models(d.h, None))
    d.close()
    prof = profiler.OnlineProfiler(base, prior=[], period_steps=4)
    ctl = serving.ModeController(abi.MODE_VSD_AD, 22, fixed_k=4, models=m0, profiler=prof)
    f = profiler.serial_factor(base["draft"])
    for i in range(16):
        b, k = (1, 8, 32)[i % 3], (2, 4, 6, 8)[i % 4]
        dm, vm = synth(b, k, f)
        ctl.observe([], b, dm + vm, ks=[k] * b, draft_ms=dm, verify_ms=vm)
        if prof.future is not None:
            prof.future.result()
    assert prof.refreshes >= 1
    # one speculative length only: the load forms are not identifiable, the stages keep theirs
    m1, _ = profiler.fit_serial([{"b": b, "s": 4, "draft_ms": 1.0 + b, "verify_ms": 2.0 + b} for b in (1, 2, 3)], base)
    assert m1["target"]["c2"] == base["target"]["c2"] and m1["draft"]["c1"] == base["draft"]["c1"]
    assert ctl.models is not m0 and ctl.models.target.c2 == pytest.approx(TRUE["target"][2], rel=1e-6)
    ctl.close()

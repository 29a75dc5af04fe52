"""CPU tier: host-side scalar controllers (exitctl / overlap / latmodel eval / synth_prompt)
of the product library against the reference TUs (oracle/_ref), bit-exact."""
import ctypes as C
import os
import random

import pytest

from oracle import pyoracle as po
from paper_2604_20503_b200 import abi, engine

needs_ref = pytest.mark.skipif(not os.path.exists(po.REF_SO), reason="oracle/_ref not built")


def test_k_table_matches_oracle_k_at():
    P = po.restated()
    rng = random.Random(1)
    for _ in range(200):
        pol = abi.ExitPolicy(rng.randint(-2, 40), rng.randint(1, 30), 1)
        pol.k_final = rng.randint(1, pol.k_init)
        L = rng.randint(1, 128)
        t = engine.k_table(pol, L)
        assert [t[l] for l in range(L + 1)] == [P.k_at(pol, l, L) for l in range(L + 1)]


def test_k_table_rejects_bad_policy():
    with pytest.raises(engine.FaserError):
        engine.k_table(abi.ExitPolicy(8, 2, 10), 32)


@needs_ref
def test_gate_plan_matches_reference():
    R = po.ref()
    rng = random.Random(2)
    for _ in range(300):
        n = rng.randint(0, 40)
        ents = [(rng.choice(abi.S_CANDIDATES), rng.random()) for _ in range(n)]
        pol = abi.ExitPolicy(rng.randint(1, 40), 10, 2)
        b = float(rng.choice([1, 4, 16, 32, 64, 256]))
        r = rng.choice([0.1, 0.2, 0.5, 0.8, 0.9])
        L = rng.choice([16, 32, 80])
        g = engine.make_gate_plan(pol, ents, b, r, L)
        arr = (abi.GateEntry * max(n, 1))(*[abi.GateEntry(s, 0, a) for s, a in ents])
        ref = abi.GatePlan()
        assert R.lib.specref_make_gate_plan(C.byref(pol), arr, n, C.c_double(b), C.c_double(r), L,
                                            C.byref(ref)) == 0
        assert (g.first_layer, g.stop_layer, g.s_eff) == (ref.first_layer, ref.stop_layer, ref.s_eff)


@needs_ref
def test_gate_plan_throws_like_reference_at_r_1():
    # should_prune throws for r in {0, 1} (latmodel.cpp:45) — SURVEY Appendix A.8
    with pytest.raises(engine.FaserError) as ei:
        engine.make_gate_plan(abi.ExitPolicy.default(), [(4, 0.5)], 32.0, 1.0, 32)
    assert ei.value.status == abi.EINVAL


@needs_ref
def test_plan_overlap_matches_reference():
    R = po.ref()
    L = engine.lib()
    grid = (C.c_double * 9)(*[i / 10 for i in range(1, 10)])
    for s in range(1, 11):
        for b in (1, 2, 4, 8, 16, 32, 64, 128, 256):
            a, r = abi.OverlapPlan(), abi.OverlapPlan()
            assert L.faser_plan_overlap(s, b, None, grid, 9, C.byref(a)) == 0
            assert R.lib.specref_plan_overlap(s, b, grid, 9, C.byref(r)) == 0
            assert (a.enabled, a.chunk, a.r, a.predicted_ms, a.serial_ms) == \
                   (r.enabled, r.chunk, r.r, r.predicted_ms, r.serial_ms)


@needs_ref
def test_eval_latency_matches_reference():
    R = po.ref()
    L = engine.lib()
    for stage in range(4):
        for b in (1, 16, 256):
            for s in (1, 4, 10):
                for r in (0.1, 0.5, 0.9):
                    a, ref = C.c_double(), C.c_double()
                    assert L.faser_eval_latency(None, stage, C.c_double(b), C.c_double(s),
                                                C.c_double(r), C.byref(a)) == 0
                    assert R.lib.specref_eval_latency(stage, C.c_double(b), C.c_double(s),
                                                      C.c_double(r), C.byref(ref)) == 0
                    assert a.value == ref.value


def test_synth_prompt_matches_oracle():
    import numpy as np
    L = engine.lib()
    P = po.restated()
    for idx in range(40):
        for ln in (0, 1, 8, 100):
            out = np.zeros(max(ln, 1), np.int32)
            assert L.faser_synth_prompt(C.c_uint64(1), idx, ln, 64, out.ctypes.data_as(C.c_void_p)) == 0
            assert out.tolist() == P.synth_prompt(1, idx, ln, 64)


def _segments(L, fn_prefix, mean, ptv, dur, steps):
    import numpy as np
    d, r = np.zeros(steps), np.zeros(steps)
    rc = getattr(L, fn_prefix + "sine_segments")(C.c_double(mean), C.c_double(ptv), C.c_double(dur), steps,
                                                  d.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p))
    assert rc == 0
    return d, r


@needs_ref
@pytest.mark.parametrize("mean,ptv,dur,steps,seed", [(26.0, 10.0, 60000.0, 12, 1), (5.0, 1.0, 2000.0, 1, 7),
                                                      (100.0, 3.0, 3000.0, 7, 123)])
def test_sine_segments_and_synth_workload_match_reference(mean, ptv, dur, steps, seed):
    """Bursty config-4 arrivals (workload.cpp:73-114) bit-exact against the reference TUs."""
    import numpy as np
    L = engine.lib()
    R = po.ref().lib
    d, r = _segments(L, "faser_", mean, ptv, dur, steps)
    d2, r2 = _segments(R, "specref_", mean, ptv, dur, steps)
    assert d.tobytes() == d2.tobytes() and r.tobytes() == r2.tobytes()
    cap = 20000
    outs = []
    for lib, pre in ((L, "faser_"), (R, "specref_")):
        a, i, o, n = np.zeros(cap), np.zeros(cap, np.int32), np.zeros(cap, np.int32), C.c_int32()
        rc = getattr(lib, pre + "synth_workload")(
            d.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p), steps, 128, 1024, 64, 256,
            C.c_uint64(seed), a.ctypes.data_as(C.c_void_p), i.ctypes.data_as(C.c_void_p),
            o.ctypes.data_as(C.c_void_p), cap, C.byref(n))
        assert rc == 0
        outs.append((a[:n.value].tobytes(), i[:n.value].tolist(), o[:n.value].tolist()))
    assert outs[0] == outs[1] and len(outs[0][1]) > 0


def test_synth_workload_rejects_bad_input():
    import numpy as np
    L = engine.lib()
    d, r = np.array([-1.0]), np.array([1.0])
    n = C.c_int32()
    assert L.faser_synth_workload(d.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p), 1, 1, 2, 1, 2,
                                  C.c_uint64(1), None, None, None, 0, C.byref(n)) == abi.EINVAL

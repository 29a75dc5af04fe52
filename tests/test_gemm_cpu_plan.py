"""The sweep-driven GEMM planner (tc_gemm.cu gemm_plan_table) on the CPU: valid, instantiated
plans for any shape, deterministic, and the measured rule table kept for the configs' shapes."""
import ctypes as C

import pytest

from paper_2604_20503_b200 import engine


def _lib():
    L = engine.lib()
    L.faser_k_gemm_plan_table.argtypes = [C.c_int32] * 3 + [C.POINTER(C.c_int32), C.POINTER(C.c_double)]
    return L


@pytest.mark.parametrize("n_out,k", [(9216, 3072), (3072, 8192), (5120, 4096), (22016, 4096), (1024, 1024),
                                     (640, 2560), (49152, 6144)])
@pytest.mark.parametrize("t", [1, 7, 32, 100, 128, 300, 512, 1500, 4096])
def test_table_plan_is_an_instantiated_launch(n_out, k, t):
    L = _lib()
    o = (C.c_int32 * 4)()
    sc = C.c_double()
    assert L.faser_k_gemm_plan_table(n_out, t, k, o, C.byref(sc)) == 0
    bn, splits, mc, deep = list(o)
    assert bn in (32, 64, 128, 256) and mc in (1, 2, 4) and deep in (0, 1)
    assert mc * bn <= 512 and not (bn > 128 and mc > 2) and (mc == 1 or deep == 1)
    assert mc == 1 or n_out // 128 >= mc
    kb = k // 64
    assert 1 <= splits <= 8
    if splits > 1:
        kps = (kb + splits - 1) // splits
        assert kps >= 4 and (kb + kps - 1) // kps == splits
    assert sc.value >= 0.0
    o2 = (C.c_int32 * 4)()
    assert L.faser_k_gemm_plan_table(n_out, t, k, o2, None) == 0 and list(o2) == list(o)  # cached, same


def test_engine_uses_table_outside_measured_shapes():
    L = _lib()
    for n_out, t, k in [(9216, 128, 3072), (22016, 512, 4096)]:
        a, b = (C.c_int32 * 4)(), (C.c_int32 * 4)()
        assert L.faser_k_gemm_plan(n_out, t, k, a) == 0
        assert L.faser_k_gemm_plan_table(n_out, t, k, b, None) == 0
        assert list(a) == list(b)

"""K1/K2 projection GEMM (tcgen05 + TMEM + TMA, swap-AB, split-K) vs a torch fp32 reference
of the same op on the same bf16 operands."""
import ctypes as C

import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not has_gpu():
        pytest.skip("no GPU")
    from paper_2604_20503_b200 import engine
    return engine.lib()


# (n_out, T, K): the config-3/4 projection shapes at verify / draft row counts
SHAPES = [
    (128, 1, 64), (256, 5, 128), (2560, 20, 2048), (2048, 33, 2048), (11264, 160, 2048),
    (2048, 64, 5632), (32000, 17, 2048), (2304, 256, 768), (768, 300, 3072), (6144, 129, 768),
    (4096, 1280, 4096), (1024, 700, 1024),
]


@pytest.mark.parametrize("n_out,T,K", SHAPES)
@pytest.mark.parametrize("splits,mc", [(0, 0), (1, 1), (3, 1), (1, 2), (5, 2), (2, 4), (8, 4)])
def test_gemm_matches_fp32(L, n_out, T, K, splits, mc):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n_out * 7 + T * 3 + K)
    w = (torch.randn(n_out, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(T, K, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((T, n_out), float("nan"), device="cuda", dtype=torch.float32)
    rc = L.faser_k_gemm_bf16_plan(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()),
                                  C.c_void_p(out.data_ptr()), n_out, T, K, 10000 * mc, splits, None)
    assert rc == 0
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item()
    # fp32 accumulation of exact bf16 products: only summation order differs
    assert err <= 1e-4 * max(scale, 1.0) + 1e-3, (err, scale)


def test_gemm_rejects_bad_shapes(L):
    assert L.faser_k_gemm_bf16(C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), 100, 4, 64, 0, None) == 1
    assert L.faser_k_gemm_bf16(C.c_void_p(1), C.c_void_p(1), C.c_void_p(1), 128, 4, 60, 0, None) == 1


# the launch shapes the single-prompt prefill plan picks (gemm_plan_prefill, 256..1023 rows)
@pytest.mark.parametrize("n_out,T,K,code,splits", [
    (11264, 576, 2048, 20256, 1),   # gate/up: 256 x 256 per CTA
    (2560, 576, 2048, 128, 1),      # qkv: one 128-row token tile
    (768, 576, 3072, 128, 4),       # draft down: 4-way split
    (2048, 300, 5632, 20256, 2),    # 256 x 256 with a split
    (4096, 128, 14336, 128, 4),     # config-4 down at 128 rows
    (6144, 128, 4096, 64, 1),       # config-4 qkv
    (128256, 32, 2048, 40032, 1),   # config-4 draft LM head: 4 weight tiles per rows tile
    (28672, 128, 4096, 20128, 1),   # config-4 gate/up
])
def test_gemm_prefill_shapes_match_fp32(L, n_out, T, K, code, splits):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n_out + T + K)
    w = (torch.randn(n_out, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(T, K, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((T, n_out), float("nan"), device="cuda", dtype=torch.float32)
    assert L.faser_k_gemm_bf16_plan(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
                                    n_out, T, K, code, splits, None) == 0
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    assert (out - ref).abs().max().item() <= 1e-4 * max(ref.abs().max().item(), 1.0) + 1e-3


def _check_plan(L, n_out, T, K, code, splits):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n_out * 5 + T + K + code)
    w = (torch.randn(n_out, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(T, K, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((T, n_out), float("nan"), device="cuda", dtype=torch.float32)
    assert L.faser_k_gemm_bf16_plan(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
                                    n_out, T, K, code, splits, None) == 0
    torch.cuda.synchronize()
    ref = x.float() @ w.float().t()
    assert not torch.isnan(out).any()
    assert (out - ref).abs().max().item() <= 1e-4 * max(ref.abs().max().item(), 1.0) + 1e-3


# pipeline-depth variants the plan rules select (1000 + bn = shallow: 4 stages at 64-wide tiles,
# 3 at 128-wide; 2000 + bn = deep), with and without a K split, at production row counts
@pytest.mark.parametrize("code", [1032, 1064, 1128, 1256, 2064, 2128, 2256, 21064, 21128])
@pytest.mark.parametrize("n_out,T,K,splits", [(11264, 96, 2048, 1), (2048, 160, 5632, 4), (2560, 1000, 2048, 0),
                                              (6144, 48, 768, 1), (2048, 192, 2048, 3)])
def test_gemm_pipeline_variants_match_fp32(L, code, n_out, T, K, splits):
    _check_plan(L, n_out, T, K, code, splits)


# planner-driven launches at the exact shapes of the config-3 plan rules (tc_gemm.cu gemm_plan)
@pytest.mark.parametrize("n_out,T,K", [(2048, 192, 2048), (11264, 96, 2048), (2560, 320, 2048), (6144, 48, 768),
                                       (2560, 1000, 2048), (11264, 128, 2048), (2048, 128, 5632), (2560, 128, 2048),
                                       (32000, 128, 2048), (11264, 576, 2048), (2048, 1024, 5632), (11264, 1024, 2048),
                                       (2560, 768, 2048), (2048, 512, 5632), (11264, 512, 2048)])
def test_gemm_planner_rule_shapes_match_fp32(L, n_out, T, K):
    _check_plan(L, n_out, T, K, 0, 0)

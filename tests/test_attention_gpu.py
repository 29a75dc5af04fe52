"""K3 paged varlen causal attention (mma.sync bf16) vs a torch fp32 reference of the same op on
the same bf16 inputs (tolerance: bf16 rounding of P and O)."""
import ctypes as C

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not has_gpu():
        pytest.skip("no GPU")
    from paper_2604_20503_b200 import engine
    return engine.lib()


def run_case(L, n_q, n_kv, hd, rows_per_req, ctx, seed=0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_req = len(rows_per_req)
    max_pages = max((c + 63) // 64 for c in ctx) + 1
    n_pages = n_req * max_pages
    perm = torch.randperm(n_pages, generator=g, device="cuda").to(torch.int32)  # scattered pages
    ptab = perm.view(n_req, max_pages).contiguous()
    kv = (torch.randn(n_pages, n_kv, 2, 64, hd, device="cuda", generator=g)).to(torch.bfloat16)
    first = np.cumsum([0] + rows_per_req[:-1]).astype(np.int32)
    rows = int(sum(rows_per_req))
    q = torch.randn(rows, n_q, hd, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.zeros(rows, n_q, hd, device="cuda", dtype=torch.bfloat16)
    pos0 = [c - n for c, n in zip(ctx, rows_per_req)]  # the block's last row sees ctx keys
    t = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    d_first, d_n, d_pos0 = t(first.tolist()), t(rows_per_req), t(pos0)
    scratch = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    rc = L.faser_k_attention(C.c_void_p(q.data_ptr()), C.c_void_p(kv.data_ptr()), C.c_void_p(ptab.data_ptr()),
                             max_pages, n_req, C.c_void_p(d_first.data_ptr()), C.c_void_p(d_n.data_ptr()),
                             C.c_void_p(d_pos0.data_ptr()), max(rows_per_req), max(ctx), n_q, n_kv, hd,
                             C.c_void_p(out.data_ptr()), C.c_void_p(scratch.data_ptr()), scratch.numel(), None)
    assert rc == 0
    torch.cuda.synchronize()
    G = n_q // n_kv
    for i in range(n_req):
        pages = ptab[i].long()
        K = kv[pages, :, 0].permute(1, 0, 2, 3).reshape(n_kv, -1, hd)[:, :ctx[i]].float()
        Vv = kv[pages, :, 1].permute(1, 0, 2, 3).reshape(n_kv, -1, hd)[:, :ctx[i]].float()
        Q = q[first[i]:first[i] + rows_per_req[i]].float()  # [r][n_q][hd]
        for h in range(n_q):
            s = Q[:, h] @ K[h // G].t() / hd ** 0.5  # [r][ctx]
            pos = torch.arange(rows_per_req[i], device="cuda") + pos0[i]
            mask = torch.arange(ctx[i], device="cuda")[None, :] > pos[:, None]
            s[mask] = -float("inf")
            ref = torch.softmax(s, -1) @ Vv[h // G]
            got = out[first[i]:first[i] + rows_per_req[i], h].float()
            err = (got - ref).abs().max().item()
            assert err < 3e-2, (i, h, err)


# "batch": enough (request, kv head) units that no KV split is wanted (GQA groups of >= 4 heads
# with > 32 packed rows take the tcgen05 kernel, llama_attn_tc.cu): odd / even page counts,
# 1..1500 keys
BATCH_ROWS = [4] * 20 + [1, 2, 3, 5, 8, 4, 4, 4]
BATCH_CTX = [4, 63, 64, 65, 127, 128, 129, 191, 192, 193, 255, 256, 257, 600, 640, 700, 900, 1000, 1280, 1500,
             1, 2, 70, 300, 64, 130, 500, 777]


@pytest.mark.parametrize("n_q,n_kv,hd", [(32, 4, 64), (12, 12, 64), (32, 8, 128), (8, 8, 128)])
@pytest.mark.parametrize("shape", ["decode", "verify", "prefill", "ragged", "batch", "long", "pair", "decode_long"])
def test_attention_matches_fp32(L, n_q, n_kv, hd, shape):
    rows, ctx = {
        "decode": ([1] * 6, [1, 63, 64, 65, 300, 1000]),
        "verify": ([4, 5, 1, 10, 3], [5, 200, 640, 77, 1500]),
        "prefill": ([96, 33], [96, 33]),
        "ragged": ([2, 70, 1, 16], [2, 900, 129, 16]),
        "batch": (BATCH_ROWS, BATCH_CTX),
        "long": ([4, 4, 1], [1600, 2000, 1800]),  # few units, long contexts: the split-KV path
        "pair": ([4] * 8, [600, 700, 400, 690, 500, 640, 385, 650]),  # cluster-pair split (DSMEM merge)
        "decode_long": ([1] * 5, [1, 64, 257, 1300, 2000]),  # one row per request, 1..2000 keys
    }[shape]
    if shape == "batch" and n_q // n_kv * max(rows) > 64:
        rows = [min(r, 64 // (n_q // n_kv)) for r in rows]
    run_case(L, n_q, n_kv, hd, rows, ctx, seed=n_q + hd)


@pytest.mark.parametrize("n_q,n_kv,hd", [(32, 4, 64), (32, 8, 128), (12, 12, 64)])
@pytest.mark.parametrize("kernels", ["tcgen05", "mma_sync"])
def test_attention_dispatch_variants(n_q, n_kv, hd, kernels):
    """The non-default dispatches (env read once per process, so in a subprocess): tcgen05 for
    every GQA-packed GROUP shape (FASER_ATTN_TC=1), or the mma.sync kernels everywhere
    (FASER_ATTN_TC=0, FASER_ATTN_TC_ROWS=0)."""
    import os
    import subprocess
    import sys
    env = {"tcgen05": {"FASER_ATTN_TC": "1"},
           "mma_sync": {"FASER_ATTN_TC": "0", "FASER_ATTN_TC_ROWS": "0"}}[kernels]
    code = ("import sys; sys.path.insert(0, 'tests'); import test_attention_gpu as t; "
            "from paper_2604_20503_b200 import engine; L = engine.lib(); "
            f"t.run_case(L, {n_q}, {n_kv}, {hd}, t.BATCH_ROWS, t.BATCH_CTX, seed=5); "
            f"t.run_case(L, {n_q}, {n_kv}, {hd}, [96, 33], [96, 33], seed=6); "
            f"t.run_case(L, {n_q}, {n_kv}, {hd}, [2, 70, 1, 16], [2, 900, 129, 16], seed=7)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]

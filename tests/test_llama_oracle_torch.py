"""CPU tier: pins the builder-written fp32 Llama oracle (oracle/llama_oracle.c) against an
INDEPENDENT forward written here in torch float64 on the same weights.

The reference has no transformer, so nothing in /root/reference can pin the
Llama oracle. This test is the independent cross-check the round-1 verdict asked for: the
architecture is restated from its definition, not from the C loops —
  x_0 = emb[tok];  per layer:  x += Wo · attn(rope(Wq·n(x)), rope(Wk·n(x)), Wv·n(x))
                                x += Wd · (silu(Wg·n(x)) * (Wu·n(x)))
  logits_l = W_lm · n(x_l)          n(x) = x / sqrt(mean(x²) + eps)   (RMSNorm, gamma = 1)
with RoPE rotate-half (angle = pos · theta^(-2i/hd)), causal GQA (q head h reads kv head
h // (n_q / n_kv)), gate/up rows interleaved in groups of 64 (HBM layout) — in
float64 with torch's own matmul/softmax, against the C oracle's fp32 loops.
Tolerance: max |oracle − torch| ≤ 1e-4 × (max − min) of the torch row, at every requested layer.
"""
import numpy as np
import pytest
import torch

from oracle import lmoracle
from paper_2604_20503_b200 import llama

TOL = 1e-4


def bf16_to_f64(u16):
    return torch.from_numpy(u16.astype(np.uint32) << 16).view(torch.float32).to(torch.float64)


def torch_forward(om, tokens, layers):
    """Independent float64 forward of the oracle model `om` (weights read as whole tensors)."""
    s = om.shape
    d, nq, nkv, hd, F = s.d_model, s.n_heads, s.n_kv_heads, s.head_dim, s.ffn
    n = len(tokens)
    emb = bf16_to_f64(om.tensor(1))
    lm = bf16_to_f64(om.tensor(0))
    x = emb[torch.tensor(tokens)]
    pos = torch.arange(n, dtype=torch.float64)
    inv = torch.tensor([s.rope_theta ** (-(2.0 * i) / hd) for i in range(hd // 2)], dtype=torch.float64)
    ang = pos[:, None] * inv[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def norm(v):
        return v / torch.sqrt((v * v).mean(-1, keepdim=True) + s.rms_eps)

    def rope(t):  # [n][heads][hd]
        a, b = t[..., :hd // 2], t[..., hd // 2:]
        c, sn = cos[:, None, :], sin[:, None, :]
        return torch.cat([a * c - b * sn, b * c + a * sn], -1)

    mask = torch.full((n, n), float("-inf"), dtype=torch.float64).triu(1)
    out = {}
    for l in range(s.layers):
        wqkv = bf16_to_f64(om.tensor(2, l))
        wo = bf16_to_f64(om.tensor(3, l))
        wgu = bf16_to_f64(om.tensor(4, l)).view(F // 64, 2, 64, d)
        wg, wu = wgu[:, 0].reshape(F, d), wgu[:, 1].reshape(F, d)
        wd = bf16_to_f64(om.tensor(5, l))
        qkv = norm(x) @ wqkv.T
        q = rope(qkv[:, :nq * hd].view(n, nq, hd))
        k = rope(qkv[:, nq * hd:(nq + nkv) * hd].view(n, nkv, hd))
        v = qkv[:, (nq + nkv) * hd:].view(n, nkv, hd)
        rep = nq // nkv
        k = k.repeat_interleave(rep, dim=1)
        v = v.repeat_interleave(rep, dim=1)
        sc = torch.einsum("qhd,khd->hqk", q, k) / np.sqrt(hd) + mask
        o = torch.einsum("hqk,khd->qhd", torch.softmax(sc, -1), v).reshape(n, nq * hd)
        x = x + o @ wo.T
        h = norm(x)
        g, u = h @ wg.T, h @ wu.T
        x = x + (g * torch.sigmoid(g) * u) @ wd.T
        if l + 1 in layers:
            out[l + 1] = (norm(x) @ lm.T).numpy()
    return out


@pytest.mark.parametrize("preset,n,layers", [
    ("tiny", 40, [1, 2, 3, 4]),
    ("tiny128", 33, [1, 2, 3]),
    ("cfg3", 48, [2, 8, 16, 22]),
])
def test_c_oracle_matches_independent_torch_forward(preset, n, layers):
    desc = llama.PRESETS[preset]()
    rng = np.random.default_rng(7)
    for shape in (desc.target, desc.draft):
        lay = [l for l in layers if l <= shape.layers] or [shape.layers]
        tok = rng.integers(0, shape.vocab - 1, size=n).tolist()
        om = lmoracle.Model(shape, desc.bigram_a, desc.bigram_b)
        got = om.logits(tok, 0, lay)
        ref = torch_forward(om, tok, set(lay))
        om.close()
        for i, l in enumerate(lay):
            r = ref[l]
            rng_row = r.max(-1) - r.min(-1)
            err = (np.abs(got[i].astype(np.float64) - r).max(-1) / rng_row).max()
            assert err <= TOL, (preset, shape.d_model, l, err)
            assert (got[i].argmax(-1) == r.argmax(-1)).mean() >= 0.99

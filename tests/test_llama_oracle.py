"""CPU tier: the Llama-path oracle itself (test infrastructure) — its weight generator against an
independent pure-Python restatement, and the oracle SD loop's losslessness (the reference's
master property) on the small preset."""
import numpy as np

from oracle import lmoracle, lmsd
from paper_2604_20503_b200 import abi, llama

M64 = (1 << 64) - 1


def mix64(x):
    return abi.mix64(x & M64)


def py_gen(seed, tag, i, std):
    """Pure-Python restatement of gen_value (llama_oracle.c / llama_kernels.cu)."""
    base = mix64(seed ^ mix64(tag))
    r = mix64((base + i * 0x9E3779B97F4A7C15) & M64)
    s = (r & 0xFFFF) + ((r >> 16) & 0xFFFF) + ((r >> 32) & 0xFFFF) + (r >> 48)
    c = np.float32(np.float64(np.float32(std)) / 37837.226772)
    f = np.float32(np.float32(s - 131070) * c)
    u = int(np.array([f], np.float32).view(np.uint32)[0])
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFFFFFF
    return u >> 16


def test_weight_generator_matches_python_restatement():
    d = llama.tiny()
    m = lmoracle.Model(d.target, d.bigram_a, d.bigram_b)
    s = d.target
    for which, tag in ((0, 1 * 4096), (2, 3 * 4096 + 1), (3, 4 * 4096 + 2), (5, 7 * 4096 + 3)):
        layer = (tag % 4096)
        for i in (0, 1, 7, 1000, 12345):
            assert m.weight(which, layer, i) == py_gen(s.seed, tag, i, s.init_std)
    m.close()


def test_embedding_is_bigram_plus_noise():
    d = llama.tiny()
    m = lmoracle.Model(d.target, d.bigram_a, d.bigram_b)
    s = d.target
    V, D = s.vocab, s.d_model
    for t in (0, 5, V - 1):
        g = (d.bigram_a * t + d.bigram_b) % V
        for c in (0, 17, D - 1):
            lm = np.array([m.weight(0, 0, g * D + c) << 16], np.uint32).view(np.float32)[0]
            noise_u = py_gen(s.seed, 2 * 4096, t * D + c, s.embed_noise)  # bf16 of the noise only
            emb = np.array([m.weight(1, 0, t * D + c) << 16], np.uint32).view(np.float32)[0]
            noise = np.array([noise_u << 16], np.uint32).view(np.float32)[0]
            assert abs(emb - np.float32(s.bigram_scale) * lm) <= abs(noise) * 1.01 + abs(emb) * 2 ** -7
    m.close()


def test_oracle_sd_is_lossless_on_tiny():
    d = llama.tiny()
    sd = lmsd.OracleSD(d, threads=2)
    rng = np.random.default_rng(0)
    V = d.target.vocab
    acc = sub = 0
    for i in range(4):
        p = rng.integers(0, V - 1, size=int(rng.integers(1, 20))).tolist()
        mo = int(rng.integers(1, 30))
        sd.submit(i, p, mo)
        k = 1 + i % 5
        while not sd.reqs[i].done:
            dr, a, _, _ = sd.round(i, k)
            acc += a
            sub += len(dr)
        assert sd.reqs[i].committed == sd.target.greedy(p, mo, V - 1)
    assert 0 < acc <= sub
    sd.close()


def test_oracle_logits_layers_consistent():
    """Logits after L layers through lmo_forward equal the greedy decode's argmax path."""
    d = llama.tiny()
    m = lmoracle.Model(d.target, d.bigram_a, d.bigram_b)
    p = [1, 2, 3, 4, 5]
    g = m.greedy(p, 3, d.target.vocab - 1)
    z = m.logits(p + g[:2], len(p) - 1)[0]
    assert [int(r.argmax()) for r in z] == g
    zl = m.logits(p, 0, [1, d.target.layers])
    assert zl.shape == (2, len(p), d.target.vocab)
    m.close()

"""TEST INFRASTRUCTURE ONLY — CPU restatement of the product's coupled Gumbel-max sampling
(faser_set_sampling; tc_gemm.cu smix64 / sample_key / gumbel / perturb). The reference is
greedy only (sdcore.cpp:61-80), so this restates the product's own published rule,
not a reference algorithm ("parity unpinned" against the reference; the losslessness claim is
checked against the fp32 oracle's autoregressive sampling, tests/test_sampling_gpu.py).

Rule: the token at absolute position p of request r is argmax_v(z_v * (1/tau) + G_v) with
  key = smix64(smix64(seed) ^ (r * 0xd1b54a32d192ed03) ^ (p * 0x8cb92ba72f3d8dd7))  (mod 2^64)
  u_v = (top 23 bits of smix64(key ^ (v * 0x9e3779b97f4a7c15)) + 0.5) * 2^-23
  G_v = -log(-log(u_v))  (fp32; computed here in fp64 and rounded)
and ties to the lowest id. Only tests/, smoke() and bench.py's cpu_baseline leg may import it."""
import numpy as np

M64 = (1 << 64) - 1


def smix64(x):
    """SplitMix64 finaliser on python ints (rng.hpp:17-22 form)."""
    x = (x + 0x9e3779b97f4a7c15) & M64
    x = ((x ^ (x >> 30)) * 0xbf58476d1ce4e5b9) & M64
    x = ((x ^ (x >> 27)) * 0x94d049bb133111eb) & M64
    return x ^ (x >> 31)


def sample_key(seed, rid, pos):
    return smix64(smix64(seed & M64) ^ ((rid * 0xd1b54a32d192ed03) & M64) ^ ((pos * 0x8cb92ba72f3d8dd7) & M64))


def _smix64_np(x):
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9e3779b97f4a7c15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return x ^ (x >> np.uint64(31))


def gumbel_row(key, V, id_off=0):
    """G_v for v = id_off .. id_off + V - 1 (float32)."""
    v = np.arange(id_off, id_off + V, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _smix64_np(np.uint64(key) ^ (v * np.uint64(0x9e3779b97f4a7c15)))
    u = ((h >> np.uint64(41)).astype(np.float64) + 0.5) * 2.0 ** -23
    return (-np.log(-np.log(u))).astype(np.float32)


def perturbed(z, temperature, key):
    """z / tau + G in the device's fp32 operation order (round the product, then the sum)."""
    z = np.asarray(z, np.float32)
    inv = np.float32(1.0 / temperature)
    return (z * inv).astype(np.float32) + gumbel_row(key, z.shape[-1])


def sample(z, temperature, key):
    return int(np.argmax(perturbed(z, temperature, key)))


def sampled_decode(model, prompt, max_out, eos, rid, seed, temperature):
    """Autoregressive coupled-Gumbel sampling from the fp32 oracle model (lmoracle.Model):
    the output speculative sampling must reproduce. Returns (tokens, per-step perturbed rows)."""
    toks = list(prompt)
    out, rows = [], []
    while len(out) < max_out:
        z = model.logits(toks, len(toks) - 1)[0][0]
        y = perturbed(z, temperature, sample_key(seed, rid, len(toks)))
        t = int(np.argmax(y))
        rows.append((z, y))
        out.append(t)
        toks.append(t)
        if t == eos:
            break
    return out, rows

"""CPU tier: the coupled Gumbel-max sampling rule (oracle/sampling.py restating tc_gemm.cu's
sample_key / gumbel / perturb): the vectorised noise equals the scalar definition, and the
Gumbel-max draw is a sample of softmax(z / tau) (chi-square over many keys)."""
import math

import numpy as np

from oracle import sampling as S


def test_vectorised_noise_matches_scalar_definition():
    key = S.sample_key(7, 123456789, 42)
    g = S.gumbel_row(key, 64, id_off=1000)
    for v in (0, 1, 17, 63):
        h = S.smix64(key ^ (((1000 + v) * 0x9e3779b97f4a7c15) & S.M64))
        u = ((h >> 41) + 0.5) * 2.0 ** -23
        assert g[v] == np.float32(-math.log(-math.log(u)))
    assert 0.0 < (((S.smix64(1) >> 41) + 0.5) * 2.0 ** -23) < 1.0
    # keys differ across seed, request and position
    ks = {S.sample_key(s, r, p) for s in (0, 1) for r in (0, 1, 2**40) for p in (0, 1, 5)}
    assert len(ks) == 18


def test_gumbel_max_samples_softmax():
    z = np.array([2.0, 1.0, 0.5, 0.0, -1.0, 1.5, 0.25, -0.5], np.float32)
    for tau in (0.7, 1.0, 2.5):
        p = np.exp(z / tau - (z / tau).max())
        p /= p.sum()
        n = 20000
        cnt = np.bincount([S.sample(z, tau, S.sample_key(3, i, 9)) for i in range(n)], minlength=len(z))
        chi2 = float(((cnt - n * p) ** 2 / (n * p)).sum())
        assert chi2 < 30.0, (tau, chi2, cnt, n * p)  # 7 dof: P(chi2 > 30) ~ 1e-4


def test_temperature_limits():
    z = np.array([0.3, 2.0, 1.9, -4.0], np.float32)
    # tiny temperature -> greedy
    assert all(S.sample(z, 1e-4, S.sample_key(1, i, 2)) == 1 for i in range(200))
    # same key -> same draw (the coupling the draft and the target share)
    k = S.sample_key(5, 77, 12)
    assert S.sample(z, 1.0, k) == S.sample(z + np.float32(0.0), 1.0, k)

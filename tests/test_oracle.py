"""CPU tier: pin the oracle before trusting it.

(1) the restated C oracle (oracle/toy_oracle.c) against the REFERENCE's own TUs
(oracle/_ref, compiled in place) on seeded random inputs — bit-exact, including the
per-round VerifyOutcome records of whole serving episodes;
(2) both against the committed golden vectors (tests/golden/toy_golden.json, generated from
the reference by tests/golden/make_golden.py);
(3) the SPEC.md per-operation examples (KATs).
The reference library is built here from /root/reference; when it is absent (GPU box) the
restated oracle is still checked against the golden vectors.
"""
import os
import random

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2604_20503_b200 import abi

HAVE_REF = os.path.exists(po.REF_SO)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (no /root/reference)")


def oracles():
    out = [po.restated()]
    if HAVE_REF:
        out.append(po.ref())
    return out


def rand_prefix(rng, V, lo=1, hi=40):
    return [rng.randrange(V - 1) for _ in range(rng.randint(lo, hi))]


# ------------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
def test_golden_prompts_and_ar_decode(o, golden):
    p = abi.ToyParams.default()
    prompts = [o.synth_prompt(1, i, 8, 64) for i in range(16)]
    assert prompts == golden["synth_prompt_seed1_len8"]
    # idx0 prompt [56 45 33 62 25 24 25 3] -> AR decode(24) ends in EOS at 14
    assert prompts[0] == [56, 45, 33, 62, 25, 24, 25, 3]
    ar = [o.autoregressive_decode(p, pr, 24) for pr in prompts]
    assert ar == golden["ar_decode_24"]
    assert ar[0] == [3, 12, 56, 20, 36, 52, 8, 58, 51, 43, 43, 33, 19, 63]


@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
def test_golden_logits_bitexact(o, golden):
    p = abi.ToyParams.default()
    prompts = golden["synth_prompt_seed1_len8"][:4]
    zf, zn = o.final_and_noise(p, prompts)
    assert [[float.hex(float(x)) for x in r] for r in zf] == golden["z_final_rows0_3"]
    assert [[float.hex(float(x)) for x in r] for r in zn] == golden["z_noise_rows0_3"]
    assert zf[0, :4].tolist() == [0.10005879192559775, 0.36065013367565157, 2.7998514017584695,
                                  3.889534265188797]
    for l, row in golden["target_logits_row0"].items():
        z = o.target_logits(p, [prompts[0]], [int(l)])[0]
        assert [float.hex(float(x)) for x in z] == row


@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
def test_golden_k_at_and_agreement(o, golden):
    pol = abi.ExitPolicy.default()
    assert [o.k_at(pol, l, 32) for l in range(33)] == golden["k_at_L32"]
    # probe values quoted in SURVEY §8a row 15
    assert (o.k_at(pol, 9, 32), o.k_at(pol, 16, 32), o.k_at(pol, 24, 32), o.k_at(pol, 31, 32)) == (10, 7, 5, 2)
    pre = [o.synth_prompt(5, i, 1 + i % 24, 64) for i in range(2000)]
    for eta, rate in golden["agreement_vs_eta_2000"].items():
        q = abi.ToyParams.default(divergence=float(eta))
        assert float((o.target_next(q, pre) == o.draft_next(q, pre)).mean()) == rate


@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
@pytest.mark.parametrize("name", ["cfg1_vsd_b4_k4", "cfg1_ee_b4_k4", "cfg2_ee_b32_dyn",
                                  "cfg2_ee_b32_dyn_eta05", "b256_vsd_k4_backlog300"])
def test_golden_episodes(o, golden, name):
    import hashlib
    e = golden["episodes"][name]
    p = abi.ToyParams.default(divergence=e["divergence"])
    assert po.backlog_lengths(1, e["n"]) == (e["in_len"], e["out_len"])
    prompts = [o.synth_prompt(1, i, e["in_len"][i], 64) for i in range(e["n"])]
    cfg = abi.EpisodeCfg(model=p, max_batch=e["max_batch"], early_exit=e["early_exit"],
                         k_mode=e["k_mode"], fixed_k=e["fixed_k"], exempt_rule=1, threads=1,
                         k_seed=e["k_seed"], policy=abi.ExitPolicy.default(),
                         gate=abi.GatePlan(8, 32, 1.0))
    outs, log, st = o.run_episode(cfg, prompts, e["out_len"], log_cap=200000)
    assert outs == e["outputs"]
    for k, v in e["stats"].items():
        assert getattr(st, k) == v, k
    h = hashlib.sha256()
    for r in log:
        h.update(repr(r.as_tuple()).encode())
    assert h.hexdigest() == e["records_sha256"]
    # losslessness: every output equals the autoregressive oracle
    for pr, mo, out in zip(prompts, e["out_len"], outs):
        assert out == o.autoregressive_decode(p, pr, mo)


# ------------------------------------------------------------------ SPEC KATs
@pytest.mark.parametrize("o", oracles(), ids=lambda o: o.kind)
def test_spec_kats(o):
    # token_exit_test vs a stable-sort rank oracle on heavily tied vectors
    rng = np.random.default_rng(3)
    for _ in range(300):
        V = int(rng.integers(2, 80))
        z = rng.integers(0, 4, V).astype(np.float64)
        d = int(rng.integers(0, V))
        k = int(rng.integers(1, V + 2))
        rank = sum(1 for v in range(V) if z[v] > z[d] or (z[v] == z[d] and v < d))
        assert o.token_exit_test(z, d, k) == (rank >= k)
    # eta = 0 => draft == target; eta = 1 => token 0
    pre = [o.synth_prompt(9, i, 5 + i % 7, 64) for i in range(200)]
    p0, p1 = abi.ToyParams.default(divergence=0.0), abi.ToyParams.default(divergence=1.0)
    assert (o.draft_next(p0, pre) == o.target_next(p0, pre)).all()
    assert (o.draft_next(p1, pre) == 0).all()
    # layer L endpoint exact, midpoint = mean (SPEC.md target_logits examples)
    p = abi.ToyParams.default()
    zf, zn = o.final_and_noise(p, pre[:5])
    assert (o.target_logits(p, pre[:5], [32] * 5) == zf).all()
    assert np.allclose(o.target_logits(p, pre[:5], [16] * 5), 0.5 * zf + 0.5 * zn, rtol=0, atol=1e-15)
    assert o.autoregressive_decode(p, pre[0], 0) == []


# ------------------------------------------------------------------ restated == reference
@needs_ref
def test_restated_matches_reference_rows():
    rng = random.Random(11)
    R, P = po.ref(), po.restated()
    for trial in range(6):
        p = abi.ToyParams.default(divergence=rng.random(), seed=rng.randrange(1 << 40),
                                  noise_seed=rng.randrange(1 << 40), vocab=rng.choice([2, 7, 64, 100, 256]),
                                  layers=rng.choice([1, 4, 32, 48]), order=rng.choice([1, 2, 3, 5]))
        rows = [rand_prefix(rng, p.vocab) for _ in range(60)]
        a, b = R.final_and_noise(p, rows), P.final_and_noise(p, rows)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
        lay = [rng.randint(1, p.layers) for _ in rows]
        assert (R.target_logits(p, rows, lay) == P.target_logits(p, rows, lay)).all()
        assert (R.target_next(p, rows) == P.target_next(p, rows)).all()
        assert (R.draft_next(p, rows) == P.draft_next(p, rows)).all()
        s = [rng.randint(1, 12) for _ in rows]
        rem = [rng.randint(1, 15) for _ in rows]
        assert R.draft_tokens(p, rows, s, rem) == P.draft_tokens(p, rows, s, rem)


@needs_ref
def test_restated_matches_reference_verify():
    rng = random.Random(12)
    R, P = po.ref(), po.restated()
    for trial in range(8):
        p = abi.ToyParams.default(divergence=rng.choice([0.0, 0.3, 0.7]), layers=rng.choice([8, 32, 40]))
        n = 80
        rows = [rand_prefix(rng, 64, 1, 30) for _ in range(n)]
        committed = [rng.randint(0, len(r) - 1) for r in rows]
        # drafted = draft model continuation with random corruption (exercise mismatches)
        drafted = P.draft_tokens(p, rows, [rng.randint(1, 10) for _ in rows], [20] * n)
        drafted = [[t if rng.random() > 0.15 else rng.randrange(64) for t in d] for d in drafted]
        exempt = [c + rng.randint(0, 3) if rng.random() < 0.3 else -1 for c in committed]
        pol = abi.ExitPolicy(rng.choice([1, 4, 8]), rng.choice([3, 10, 20]), rng.choice([1, 2, 3]))
        gate = abi.GatePlan(rng.choice([0, 2, 8]), rng.choice([0, 16, 32, 64]), 1.0)
        a = R.verify(p, rows, committed, exempt, drafted, pol, gate)
        b = P.verify(p, rows, committed, exempt, drafted, pol, gate)
        assert [x.as_tuple() for x in a] == [x.as_tuple() for x in b]
        a = R.verify(p, rows, committed, exempt, drafted)
        b = P.verify(p, rows, committed, exempt, drafted)
        assert [x.as_tuple() for x in a] == [x.as_tuple() for x in b]


@needs_ref
@pytest.mark.parametrize("eta", [0.0, 0.3, 0.5, 0.7])
@pytest.mark.parametrize("ee", [0, 1])
def test_restated_matches_reference_episodes(eta, ee):
    R, P = po.ref(), po.restated()
    p = abi.ToyParams.default(divergence=eta)
    n = 100
    inl, outl = po.backlog_lengths(3, n)
    prompts = [P.synth_prompt(3, i, inl[i], 64) for i in range(n)]
    cfg = abi.EpisodeCfg(model=p, max_batch=24, early_exit=ee, k_mode=1, fixed_k=4, exempt_rule=1,
                         threads=1, k_seed=5, policy=abi.ExitPolicy.default(), gate=abi.GatePlan(8, 32, 1.0))
    o1, l1, s1 = R.run_episode(cfg, prompts, outl, log_cap=100000)
    o2, l2, s2 = P.run_episode(cfg, prompts, outl, log_cap=100000)
    assert o1 == o2
    assert [r.as_tuple() for r in l1] == [r.as_tuple() for r in l2]
    for pr, mo, out in zip(prompts, outl, o1):
        assert out == P.autoregressive_decode(p, pr, mo)


@needs_ref
def test_reference_threaded_runner_matches_single_thread():
    R = po.ref()
    p = abi.ToyParams.default()
    inl, outl = po.backlog_lengths(1, 64)
    prompts = [R.synth_prompt(1, i, inl[i], 64) for i in range(64)]
    cfg = abi.EpisodeCfg(model=p, max_batch=32, early_exit=1, k_mode=1, exempt_rule=1, threads=1,
                         k_seed=7, policy=abi.ExitPolicy.default(), gate=abi.GatePlan(8, 32, 1.0))
    o1, l1, _ = R.run_episode(cfg, prompts, outl, log_cap=100000)
    cfg.threads = 4
    o2, l2, _ = R.run_episode(cfg, prompts, outl, log_cap=100000)
    assert o1 == o2 and [r.as_tuple() for r in l1] == [r.as_tuple() for r in l2]


def test_sched_k_python_matches_c():
    import ctypes as C
    lib = po.restated().lib
    lib.oracle_sched_k.restype = C.c_int32
    for rid in range(50):
        for rnd in range(10):
            assert abi.sched_k(7, rid, rnd) == lib.oracle_sched_k(C.c_uint64(7), C.c_int64(rid), rnd)

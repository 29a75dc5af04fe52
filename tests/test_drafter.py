"""CPU tier: the native AdaptiveDrafter restatement (drafter.cpp) against a numpy restatement of
the reference's raw-window GP (drafter.cpp:46-80, Eigen LLT), its cold-start sweep
(drafter.cpp:182-186) and its LCB argmin (drafter.cpp:188-205). The reference TU needs Eigen
(absent), so this pins the controller to the reference's published algorithm, not its binary."""
import math

import numpy as np

from paper_2604_20503_b200 import abi, controller, engine

S = [1, 2, 3, 4, 5, 6, 8, 10]


def gp_reference(window, cfg):
    """drafter.cpp:46-80 with a dense solve over the raw window (what Eigen's LLT computes)."""
    m = len(S)
    if not window:
        return np.zeros(m), np.full(m, math.sqrt(cfg.kernel_var))
    idx = np.array([w[0] for w in window], float)
    y = np.array([w[1] for w in window])
    mean = y.mean()
    ls2 = 2 * cfg.kernel_len ** 2
    K = cfg.kernel_var * np.exp(-(idx[:, None] - idx[None, :]) ** 2 / ls2) + cfg.noise_var * np.eye(len(idx))
    alpha = np.linalg.solve(K, y - mean)
    mu, sd = np.zeros(m), np.zeros(m)
    for c in range(m):
        k = cfg.kernel_var * np.exp(-(c - idx) ** 2 / ls2)
        mu[c] = mean + k @ alpha
        sd[c] = math.sqrt(max(cfg.kernel_var - k @ np.linalg.solve(K, k), 1e-12))
    return mu, sd


def test_beta_and_objective():
    cfg = controller.DrafterCfg.default()
    L = engine.lib()
    for n in (0, 1, 2, 10, 1000):
        exp = 2 * math.log(8 * max(n, 1) ** 2 * math.pi ** 2 / 6)
        assert abs(L.faser_drafter_beta(cfg and __import__("ctypes").byref(cfg), n) - exp) < 1e-12
    import ctypes as C
    out = C.c_double()
    assert L.faser_drafter_objective(C.c_double(3.0), 4, C.c_double(0.5), C.c_double(1e-6), C.byref(out)) == 0
    assert abs(out.value - 3.0 / (2.0 + 1e-6)) < 1e-15
    assert L.faser_drafter_objective(C.c_double(0.0), 4, C.c_double(0.5), C.c_double(1e-6), C.byref(out)) == abi.EINVAL
    assert L.faser_drafter_objective(C.c_double(1.0), 0, C.c_double(0.5), C.c_double(1e-6), C.byref(out)) == abi.EINVAL


def test_cold_start_sweep_then_lcb():
    d = controller.AdaptiveDrafter()
    rng = np.random.default_rng(0)
    ids = list(range(6))
    seen = []
    for rnd in range(len(S)):
        k = d.assign_lengths(ids, 6, 0.5)
        assert len(set(k)) == 1
        seen.append(k[0])
        acc = [int(rng.integers(0, k[0] + 1)) for _ in ids]
        d.observe_round(6, 0.5, 1.0 + 0.1 * k[0], ids, k, k, acc)
    assert seen == S  # every arm swept once
    k = d.assign_lengths(ids, 6, 0.5)
    assert all(x in S for x in k)


def test_posterior_matches_raw_window_llt():
    cfg = controller.DrafterCfg.default()
    d = controller.AdaptiveDrafter(cfg)
    rng = np.random.default_rng(1)
    window = []  # (index, cost, round)
    b, r = 16, 0.5
    for rnd in range(1, 90):
        ks = [S[int(i)] for i in rng.integers(0, 8, size=5)]
        sub = ks
        acc = [int(rng.integers(0, k + 1)) for k in ks]
        t = float(rng.uniform(1, 5))
        d.observe_round(b, r, t, list(range(5)), ks, sub, acc)
        by_s = {}
        for k, a in zip(ks, acc):
            by_s.setdefault(k, []).append(a / k)
        for k in sorted(by_s):
            ratio = sum(by_s[k]) / len(by_s[k])
            window.append((S.index(k), t / (k * ratio + cfg.epsilon), rnd))
        window = [w for w in window if w[2] > rnd - cfg.window_ctx]
        if rnd % 11 == 0:
            mu, sd, n = d.posterior(b, r)
            emu, esd = gp_reference(window, cfg)
            assert n == rnd
            assert np.allclose(mu, emu, rtol=1e-9, atol=1e-9), (mu, emu)
            assert np.allclose(sd, esd, rtol=1e-9, atol=1e-9), (sd, esd)


def test_contexts_are_bucketed():
    d = controller.AdaptiveDrafter()
    d.observe_round(16, 0.5, 1.0, [0], [4], [4], [2])
    assert d.posterior(17, 0.46)[2] == 1     # round(log2 17) = 4, decile 5: same context
    assert d.posterior(64, 0.5)[2] == 0
    assert d.posterior(16, 0.9)[2] == 0


def test_rejects_unknown_length():
    d = controller.AdaptiveDrafter()
    try:
        d.observe_round(4, 0.5, 1.0, [0], [7], [7], [3])
    except engine.FaserError as e:
        assert e.status == abi.EINVAL
    else:
        raise AssertionError("7 is not in the candidate set")


def test_request_window_pinned_to_reference_acceptance_window():
    """The drafter's per-request window (drafter.cpp ReqWindow) against the reference's OWN
    AcceptanceWindow (sdcore.cpp:8-35, compiled in place in oracle/_ref): the same rounds pushed
    through both, rate_for(s) for every s in S and overall() compared bit-for-bit after every
    push, across the W = 16 eviction boundary and with submitted = 0 rounds."""
    import ctypes as C
    import os

    import pytest

    from oracle import pyoracle as po
    if not os.path.exists(po.REF_SO):
        pytest.skip("oracle/_ref not built")
    R = po.ref().lib
    rng = np.random.default_rng(12)
    n = 40
    s = rng.choice(S, size=n).astype(np.int32)
    sub = np.minimum(s, rng.integers(0, 11, size=n)).astype(np.int32)
    sub[[3, 17]] = 0
    acc = np.array([rng.integers(0, x + 1) for x in sub], np.int32)
    qs = np.array(S, np.int32)
    cfg = controller.DrafterCfg.default()
    ref = np.zeros((n, len(S) + 1))
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert R.specref_acceptance_window_replay(p(s), p(sub), p(acc), n, cfg.window_request, p(qs), len(S),
                                              p(ref)) == 0
    d = controller.AdaptiveDrafter()
    for i in range(n):
        d.observe_round(1, 1.0, 1.0, [7], [int(s[i])], [int(sub[i])], [int(acc[i])])
        got = d.request_window(7, S)
        assert got == ref[i].tolist(), i
    d.close()


def test_estimate_fallback_chain():
    """AcceptanceBook::estimate (drafter.cpp:151-161): request window rate for s, then the
    context's rate for s, then the context overall, then the request overall, then cold start."""
    cfg = controller.DrafterCfg.default()
    d = controller.AdaptiveDrafter()
    assert d.estimate([1], [4], 8, 1.0) == [cfg.cold_start_accept]
    d.observe_round(8, 1.0, 1.0, [1, 2], [4, 2], [4, 2], [3, 1])
    a = d.estimate([1, 2, 1, 3], [4, 4, 2, 5], 8, 1.0)
    assert a[0] == 0.75          # request 1's own window at s = 4
    assert a[1] == 0.75          # request 2 has no s = 4 round: the context's rate for s = 4
    assert a[2] == 0.5           # request 1 has no s = 2 round: the context's rate for s = 2
    assert a[3] == (0.75 + 0.5) / 2  # nobody ran s = 5: the context overall
    d.close()


def test_drafter_matches_reference_translation_unit():
    """The native AdaptiveDrafter (csrc/drafter.cpp) against the REFERENCE's own drafter.cpp,
    compiled in place into oracle/_ref with oracle/eigen_shim standing in for its three Eigen
    calls (MatrixXd / VectorXd / LLT solve): same k_i assignments round by round (cold-start
    sweep, then GP-LCB with the AcceptanceBook estimates and the latency lanes) and the same GP
    posterior to rounding, over a random serving history in two (b, r) contexts."""
    import ctypes as C
    import os

    import pytest

    from oracle import pyoracle as po
    from paper_2604_20503_b200 import llama
    if not os.path.exists(po.REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    L = C.CDLL(po.REF_SO)
    if not hasattr(L, "specref_drafter_create"):
        pytest.skip("oracle/_ref predates the drafter export")
    L.specref_drafter_create.restype = C.c_void_p
    L.specref_drafter_create.argtypes = [C.c_void_p, C.c_void_p]
    L.specref_drafter_destroy.argtypes = [C.c_void_p]
    L.specref_drafter_assign.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_void_p]
    L.specref_drafter_observe.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int32]
    L.specref_drafter_posterior.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    cfg = controller.DrafterCfg.default()
    for models in (None, llama.fitted_latency_model()):
        nat = controller.AdaptiveDrafter(cfg, models=models)
        ref = L.specref_drafter_create(C.byref(cfg), C.byref(models) if models is not None else None)
        rng = np.random.default_rng(7)
        pool = np.arange(100, 140, dtype=np.int64)
        mism = 0
        for rnd in range(160):
            b = int(rng.choice([4, 16]))
            r = float(rng.choice([1.0, 0.5]))
            live = np.sort(rng.choice(pool, size=b, replace=False)).astype(np.int64)
            kn = np.array(nat.assign_lengths(live, b, r), np.int32)
            kr = np.zeros(b, np.int32)
            assert L.specref_drafter_assign(ref, P(live), b, b, r, P(kr)) == 0
            mism += int((kn != kr).sum())
            spec = kn
            sub = np.minimum(spec, rng.integers(1, 11, size=b)).astype(np.int32)
            acc = np.array([rng.integers(0, s + 1) for s in sub], np.int32)
            t = float(rng.uniform(1.0, 6.0))
            nat.observe_round(b, r, t, live, spec, sub, acc)
            assert L.specref_drafter_observe(ref, b, r, t, P(live), P(spec), P(sub), P(acc), b) == 0
            mu_n, sd_n, rn = nat.posterior(b, r)
            mu_r, sd_r = np.zeros(cfg.n_candidates), np.zeros(cfg.n_candidates)
            rr = C.c_int32()
            L.specref_drafter_posterior(ref, b, r, P(mu_r), P(sd_r), C.byref(rr))
            assert rn == rr.value
            np.testing.assert_allclose(mu_n, mu_r, rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(sd_n, sd_r, rtol=1e-9, atol=1e-9)
        assert mism == 0, f"{mism} k_i assignments differ from the reference drafter"
        L.specref_drafter_destroy(ref)
        nat.close()

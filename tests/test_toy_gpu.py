"""GPU tier (B200): the CUDA toy path against the CPU oracle, bit-exact.

Every call goes through the C ABI (libfaser_b200.so). Checked against the restated oracle
(oracle/_build) and, where the prebuilt reference library travelled with the snapshot
(oracle/_ref), against the reference's own TUs; episode round logs are also checked
against the committed golden fixtures generated from the reference.
"""
import hashlib
import os
import random

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2604_20503_b200 import abi, engine, serving

pytestmark = pytest.mark.gpu


def checkers():
    out = [po.restated()]
    if os.path.exists(po.REF_SO):
        out.append(po.ref())
    return out


def rand_prefix(rng, V, lo=1, hi=40):
    return [rng.randrange(V - 1) for _ in range(rng.randint(lo, hi))]


PARAMS = [
    abi.ToyParams.default(),
    abi.ToyParams.default(divergence=0.7, seed=123456789, noise_seed=99, vocab=200, layers=48, order=3),
    abi.ToyParams.default(divergence=0.0, vocab=2, layers=1, order=1),
    abi.ToyParams.default(divergence=0.5, vocab=33, layers=8, order=5, logit_scale=0.25, noise_scale=3.0),
    abi.ToyParams.default(divergence=1.0, vocab=256, layers=128, order=2),
]


@pytest.mark.parametrize("pi", range(len(PARAMS)))
def test_row_ops_bitexact(pi):
    p = PARAMS[pi]
    rng = random.Random(pi)
    rows = [rand_prefix(rng, p.vocab, 1, 70) for _ in range(333)]
    toy = engine.LayeredToyLM(p)
    zf, zn = toy.final_and_noise(rows)
    lay = [rng.randint(1, p.layers) for _ in rows]
    z = toy.target_logits(rows, lay)
    tn, dn = toy.target_next(rows), toy.draft_next(rows)
    for o in checkers():
        a, b = o.final_and_noise(p, rows)
        assert (zf == a).all() and (zn == b).all()  # bit-exact doubles
        assert (z == o.target_logits(p, rows, lay)).all()
        assert (tn == o.target_next(p, rows)).all()
        assert (dn == o.draft_next(p, rows)).all()


def test_golden_logits(golden):
    p = abi.ToyParams.default()
    toy = engine.LayeredToyLM(p)
    prompts = golden["synth_prompt_seed1_len8"]
    zf, zn = toy.final_and_noise(prompts[:4])
    assert [[float.hex(float(x)) for x in r] for r in zf] == golden["z_final_rows0_3"]
    assert [[float.hex(float(x)) for x in r] for r in zn] == golden["z_noise_rows0_3"]
    for l, row in golden["target_logits_row0"].items():
        assert [float.hex(float(x)) for x in toy.target_logits([prompts[0]], int(l))[0]] == row
    pre = [po.restated().synth_prompt(5, i, 1 + i % 24, 64) for i in range(2000)]
    for eta, rate in golden["agreement_vs_eta_2000"].items():
        t = engine.LayeredToyLM(abi.ToyParams.default(divergence=float(eta)))
        assert float((t.target_next(pre) == t.draft_next(pre)).mean()) == rate


@pytest.mark.parametrize("pi", range(len(PARAMS)))
def test_draft_tokens_bitexact(pi):
    p = PARAMS[pi]
    rng = random.Random(100 + pi)
    rows = [rand_prefix(rng, p.vocab, 1, 50) for _ in range(300)]
    s = [rng.randint(1, abi.MAX_SPEC) for _ in rows]
    rem = [rng.randint(1, 40) for _ in rows]
    got = engine.SpeculativeEngine(engine.LayeredToyLM(p)).draft_tokens(rows, s, rem)
    for o in checkers():
        assert got == o.draft_tokens(p, rows, s, rem)


@pytest.mark.parametrize("pi", range(len(PARAMS)))
@pytest.mark.parametrize("gate_kind", ["full", "default", "wide", "inactive"])
def test_verify_bitexact(pi, gate_kind):
    p = PARAMS[pi]
    rng = random.Random(1000 * pi + len(gate_kind))
    n = 257
    rows = [rand_prefix(rng, p.vocab, 1, 40) for _ in range(n)]
    committed = [rng.randint(0, len(r) - 1) for r in rows]
    P = po.restated()
    drafted = P.draft_tokens(p, rows, [rng.randint(1, 12) for _ in rows], [30] * n)
    drafted = [[t if rng.random() > 0.2 else rng.randrange(p.vocab) for t in d] for d in drafted]
    exempt = [c + rng.randint(0, 4) if rng.random() < 0.3 else -1 for c in committed]
    eng = engine.SpeculativeEngine(engine.LayeredToyLM(p))
    if gate_kind == "full":
        got = eng.full_verify(rows, drafted)
        for o in checkers():
            assert [x.as_tuple() for x in got] == [x.as_tuple() for x in o.verify(p, rows, [0] * n, [-1] * n, drafted)]
        return
    pol = abi.ExitPolicy.default() if gate_kind != "wide" else abi.ExitPolicy(1, 30, 1)
    gate = {"default": abi.GatePlan(8, 32, 1.0), "wide": abi.GatePlan(0, 1000, 1.0),
            "inactive": abi.GatePlan(9, 9, 1.0)}[gate_kind]
    got = eng.verify_with_early_exit(rows, drafted, pol, gate, committed, exempt)
    for o in checkers():
        want = o.verify(p, rows, committed, exempt, drafted, pol, gate)
        assert [x.as_tuple() for x in got] == [x.as_tuple() for x in want]


def _episode_engine(p, max_batch, ee):
    return engine.ServingEngine(p, max_batch=max_batch, max_seq_len=512,
                                mode=abi.MODE_VSD_AD_EE if ee else abi.MODE_VSD)


@pytest.mark.parametrize("name", ["cfg1_vsd_b4_k4", "cfg1_ee_b4_k4", "cfg2_ee_b32_dyn",
                                  "cfg2_ee_b32_dyn_eta05", "b256_vsd_k4_backlog300"])
def test_engine_episode_matches_reference_golden(golden, name):
    e = golden["episodes"][name]
    p = abi.ToyParams.default(divergence=e["divergence"])
    P = po.restated()
    prompts = [P.synth_prompt(1, i, e["in_len"][i], 64) for i in range(e["n"])]
    with _episode_engine(p, e["max_batch"], e["early_exit"]) as eng:
        outs, recs, st = serving.run_backlog(eng, prompts, e["out_len"], k_mode=e["k_mode"],
                                             fixed_k=e["fixed_k"], k_seed=e["k_seed"],
                                             gate=abi.GatePlan(8, 32, 1.0))
        assert eng.kernel_launches() >= st["rounds"]  # one fused draft+verify+commit launch per round
    assert outs == e["outputs"]
    h = hashlib.sha256()
    for r in recs:
        h.update(repr(r).encode())
    assert len(recs) == e["n_records"]
    assert h.hexdigest() == e["records_sha256"]
    for k, v in e["stats"].items():
        assert st[k] == v, k


@pytest.mark.parametrize("eta", [0.0, 0.3, 0.5, 0.7])
@pytest.mark.parametrize("ee", [0, 1])
def test_engine_lossless_and_matches_oracle(eta, ee):
    """SPEC acceptance criterion 1 (losslessness, >=100 requests per eta, each mode) plus
    per-round record equality with the oracle's serving loop."""
    p = abi.ToyParams.default(divergence=eta)
    P = po.restated()
    n = 120
    inl, outl = po.backlog_lengths(3, n)
    prompts = [P.synth_prompt(3, i, inl[i], 64) for i in range(n)]
    with _episode_engine(p, 40, ee) as eng:
        outs, recs, _ = serving.run_backlog(eng, prompts, outl, k_mode=1, k_seed=5,
                                            gate=abi.GatePlan(8, 32, 1.0))
    cfg = abi.EpisodeCfg(model=p, max_batch=40, early_exit=ee, k_mode=1, fixed_k=4, exempt_rule=1,
                         threads=1, k_seed=5, policy=abi.ExitPolicy.default(), gate=abi.GatePlan(8, 32, 1.0))
    o2, l2, _ = P.run_episode(cfg, prompts, outl, log_cap=100000)
    assert outs == o2
    assert recs == [r.as_tuple() for r in l2]
    for pr, mo, out in zip(prompts, outl, outs):
        assert out == P.autoregressive_decode(p, pr, mo)


def test_engine_edge_cases():
    p = abi.ToyParams.default(divergence=0.4)
    P = po.restated()
    with engine.ServingEngine(p, max_batch=3, max_seq_len=256, mode=abi.MODE_VSD_AD_EE) as eng:
        # max_out = 0 is done at submission and never admitted; len-1 prompt pads the order-2
        # context with the sentinel; k > remaining clips to the budget; one long prompt.
        prompts = [[5], [7, 8], [1] * 200, [3, 4, 5], [9]]
        max_out = [0, 1, 40, 30, 50]
        outs, recs, st = serving.run_backlog(eng, prompts, max_out, fixed_k=30,
                                             gate=abi.GatePlan(8, 32, 1.0))
        for pr, mo, out in zip(prompts, max_out, outs):
            assert out == P.autoregressive_decode(p, pr, mo)
        with pytest.raises(engine.FaserError) as ei:
            eng.submit(0, [1, 2], 4)  # duplicate id
        assert ei.value.status == abi.EINVAL
        with pytest.raises(engine.FaserError) as ei:
            eng.submit(100, [64], 4)  # token outside vocab
        assert ei.value.status == abi.EINVAL
        with pytest.raises(engine.FaserError) as ei:
            eng.submit(101, [1], 1000)  # capacity
        assert ei.value.status == abi.ECAPACITY
        eng.submit(102, [1, 2, 3], 5)
        with pytest.raises(engine.FaserError):
            eng.set_spec_lengths([102], [0])
        with pytest.raises(engine.FaserError):
            eng.set_spec_lengths([102], [abi.MAX_SPEC + 1])


def test_stateless_errors_match_reference_semantics():
    eng = engine.SpeculativeEngine(engine.LayeredToyLM())
    with pytest.raises(engine.FaserError) as ei:
        eng.draft_tokens([[1, 2]], 4, 0)  # remaining 0 -> done request -> logic_error
    assert ei.value.status == abi.EILLEGAL_STATE
    with pytest.raises(engine.FaserError) as ei:
        eng.draft_tokens([[1, 2]], 0, 3)  # s < 1 -> invalid_argument
    assert ei.value.status == abi.EINVAL
    with pytest.raises(engine.FaserError) as ei:
        eng.full_verify([[1, 2]], [[]])  # empty draft
    assert ei.value.status == abi.EINVAL
    with pytest.raises(engine.FaserError) as ei:
        engine.LayeredToyLM().target_logits([[1]], 33)  # layer out of range
    assert ei.value.status == abi.EINVAL


def test_engine_max_batch_256_and_slot_reuse():
    """B_max = 256 live requests, continuous batching through 600 requests (slot reuse)."""
    p = abi.ToyParams.default()
    P = po.restated()
    n = 600
    inl, outl = po.backlog_lengths(11, n)
    prompts = [P.synth_prompt(11, i, inl[i], 64) for i in range(n)]
    with _episode_engine(p, 256, 1) as eng:
        outs, recs, st = serving.run_backlog(eng, prompts, outl, k_mode=1, k_seed=3,
                                             gate=abi.GatePlan(8, 32, 1.0))
    cfg = abi.EpisodeCfg(model=p, max_batch=256, early_exit=1, k_mode=1, fixed_k=4, exempt_rule=1,
                         threads=1, k_seed=3, policy=abi.ExitPolicy.default(), gate=abi.GatePlan(8, 32, 1.0))
    o2, l2, _ = P.run_episode(cfg, prompts, outl, log_cap=1000000)
    assert outs == o2 and recs == [r.as_tuple() for r in l2]


def test_native_serving_loop_matches_python_loop():
    """faser_serve_rounds (the sim loop in one native call) drives the engine exactly like the
    per-round Python loop with the same seeded k schedule and gate plan: identical outputs."""
    p = abi.ToyParams.default()
    P = po.restated()
    n = 48
    inl, outl = po.backlog_lengths(7, n)
    prompts = [P.synth_prompt(7, i, inl[i], 64) for i in range(n)]
    pol = abi.ExitPolicy.default()
    outs = []
    for native in (False, True):
        eng = engine.ServingEngine(p, max_batch=16, max_seq_len=256, mode=abi.MODE_VSD_AD_EE)
        for i, (pr, m) in enumerate(zip(prompts, outl)):
            eng.submit(100 + i, pr, m)
        if native:
            tok, rounds = eng.serve_rounds(10000, 7, 100, pol, 0.7, 0.5, 32)
            assert rounds > 0 and tok > 0
        else:
            rr = {}
            while eng.live_requests():
                live = eng.live_requests()
                ks = [abi.sched_k(7, rid - 100, rr.get(rid, 0)) for rid in live]
                eng.set_spec_lengths(live, ks)
                eng.set_gate(engine.make_gate_plan(pol, [(k, 0.7) for k in ks], float(len(ks)), 0.5, 32))
                for r in eng.step():
                    rr[r.req_id] = rr.get(r.req_id, 0) + 1
        outs.append([eng.committed(100 + i) for i in range(n)])
        eng.close()
    assert outs[0] == outs[1]

"""GPU tier: SM-partitioned overlap (FULL mode) — green-context lanes, frontier-chunk
cancellation, early exit inside chunks, the measured pipeline timeline and the isolated-lanes
interference baseline (overlap.cpp:44-91, overlap.hpp:11-65).

Invariant ("semantics/timing separation"): the committed token streams with overlap
on/off are identical; only the clock differs. Every finished request equals greedy decoding of
the fp32 oracle target (losslessness).
"""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import lmoracle
from paper_2604_20503_b200 import abi, engine, llama

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    if not has_gpu():
        pytest.skip("no GPU")


LOGIT_TOL = 2e-2


def check_lossless(desc, prompts, max_out, got):
    """Finished requests equal greedy decoding of the fp32 oracle; a divergence is allowed only
    where the oracle's top-2 logits are within LOGIT_TOL (bf16 vs fp32, as tests/test_llama_gpu)."""
    V = desc.target.vocab
    tgt = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b)
    for i, (p, m) in enumerate(zip(prompts, max_out)):
        ref = tgt.greedy(p, m, V - 1)
        if got[i] != ref:
            j = next(q for q in range(min(len(got[i]), len(ref))) if got[i][q] != ref[q])
            z = np.sort(tgt.logits(p + ref[:j + 1], len(p) + j - 1)[0][0])
            assert (z[-1] - z[-2]) / (z[-1] - z[0]) <= LOGIT_TOL, (i, j)
    tgt.close()


def rand_prompts(V, n, rng, lo, hi):
    return [rng.integers(0, V - 1, size=int(rng.integers(lo, hi))).tolist() for _ in range(n)]


def serve(desc, mode, prompts, max_out, k, gate=None, overlap=None, lane_mode=abi.LANES_OVERLAP, batch=4):
    eng = engine.ServingEngine(desc=desc, max_batch=batch, max_seq_len=160, mode=mode, default_spec_length=k,
                               max_spec_length=16, prefill_rows=1024)
    for i, (p, m) in enumerate(zip(prompts, max_out)):
        eng.submit(i, p, m)
    if gate is not None:
        eng.set_gate(gate)
    eng.set_lane_mode(lane_mode)
    timelines = []
    while eng.live_requests():
        if overlap:
            eng.set_overlap(True, *overlap)
        eng.step()
        if overlap:
            timelines.append(eng.last_timeline())
    out = [eng.committed(i) for i in range(len(prompts))]
    eng.close()
    return out, timelines


def check_timeline(info, evs, isolated=False):
    assert info.n_chunks >= 1
    alive = [info.chunk_alive[q] for q in range(info.n_chunks)]
    assert all(a >= b for a, b in zip(alive, alive[1:])), alive  # the frontier only shrinks
    resets = [info.chunk_resets[q] for q in range(info.n_chunks)]
    assert all(r <= a for r, a in zip(resets, alive))
    assert info.survivors + sum(resets) <= alive[0]
    d = {e.chunk: e for e in evs if e.kind == abi.EV_DRAFT_CHUNK}
    v = {e.chunk: e for e in evs if e.kind == abi.EV_VERIFY_CHUNK}
    for q, e in v.items():
        assert alive[q] > 0
        assert e.start_ms >= d[q].end_ms - 1e-3  # verify chunk q waits for draft chunk q
        if q - 1 in v:
            assert e.start_ms >= v[q - 1].end_ms - 1e-3  # verify chunks are serial on their lane
        if isolated and q + 1 in d:
            assert d[q + 1].start_ms >= e.end_ms - 1e-3  # isolated: no co-running
    for q in range(info.n_chunks):
        if alive[q] == 0:
            assert q not in v  # cancelled: nobody left to verify
    assert sum(e.kind == abi.EV_COMMIT for e in evs) == 1
    assert info.makespan_ms >= max(e.end_ms for e in evs) - 1e-6


@pytest.mark.parametrize("chunk,k,r", [(1, 4, 0.25), (2, 5, 0.5), (3, 7, 0.75)])
def test_green_lanes_full_mode_matches_serial(chunk, k, r):
    desc = llama.tiny()
    V = desc.target.vocab
    rng = np.random.default_rng(31 + chunk)
    prompts = rand_prompts(V, 6, rng, 2, 50)
    max_out = [int(rng.integers(3, 30)) for _ in range(6)]
    serial, _ = serve(desc, abi.MODE_VSD, prompts, max_out, k)
    full, tls = serve(desc, abi.MODE_FULL, prompts, max_out, k, overlap=(chunk, r))
    assert full == serial
    check_lossless(desc, prompts, max_out, full)
    info0, _ = tls[0]
    if info0.green:  # partitions of 8-SM granularity that add up to the device
        assert info0.draft_sms % 8 == 0 and info0.draft_sms >= 8
        assert info0.draft_sms + info0.verify_sms == engine.num_sms()
        lo = max(8, int(round(r * engine.num_sms() / 8)) * 8)
        assert info0.draft_sms == min(lo, (engine.num_sms() - 8) // 8 * 8)
    for info, evs in tls:
        check_timeline(info, evs)


def test_full_mode_early_exit_inside_chunks():
    """FULL = AD + EE + overlap: the gate prunes inside every frontier chunk (a prune resets the
    request's frontier, cancelling its later chunks); committed tokens equal the serial
    early-exit run's and greedy decoding of the oracle."""
    desc = llama.tiny()
    V = desc.target.vocab
    rng = np.random.default_rng(7)
    prompts = rand_prompts(V, 8, rng, 4, 60)
    max_out = [int(rng.integers(6, 40)) for _ in range(8)]
    L = desc.target.layers
    gate = abi.GatePlan(1, L, 1.0)
    serial, _ = serve(desc, abi.MODE_VSD_AD_EE, prompts, max_out, 6, gate=gate, batch=8)
    full, tls = serve(desc, abi.MODE_FULL, prompts, max_out, 6, gate=gate, overlap=(2, 0.5), batch=8)
    assert full == serial
    check_lossless(desc, prompts, max_out, full)
    resets = 0
    for info, evs in tls:
        check_timeline(info, evs)
        resets += sum(e.kind == abi.EV_RESET for e in evs)
    assert resets > 0  # frontiers were reset (rejections / prunes) and later chunks cancelled
    # some chunk had fewer requests on its frontier than the round started with
    assert any(info.chunk_alive[q] < info.chunk_alive[0] for info, _ in tls for q in range(1, info.n_chunks))


def test_isolated_lanes_same_outputs_and_no_corun():
    desc = llama.tiny()
    V = desc.target.vocab
    rng = np.random.default_rng(11)
    prompts = rand_prompts(V, 4, rng, 4, 40)
    max_out = [int(rng.integers(8, 30)) for _ in range(4)]
    a, _ = serve(desc, abi.MODE_FULL, prompts, max_out, 6, overlap=(2, 0.5))
    b, tls = serve(desc, abi.MODE_FULL, prompts, max_out, 6, overlap=(2, 0.5), lane_mode=abi.LANES_ISOLATED)
    assert a == b
    for info, evs in tls:
        assert info.lane_mode == 1
        check_timeline(info, evs, isolated=True)


def test_partitioned_single_chunk_profiles_stages():
    """chunk >= k with r in (0,1): one chunk, draft then verify on their partitions (how the
    latency profiler samples the SM-share dimension of the stage models)."""
    desc = llama.tiny()
    V = desc.target.vocab
    rng = np.random.default_rng(3)
    prompts = rand_prompts(V, 4, rng, 4, 40)
    max_out = [12] * 4
    serial, _ = serve(desc, abi.MODE_VSD, prompts, max_out, 4)
    part, tls = serve(desc, abi.MODE_FULL, prompts, max_out, 4, overlap=(4, 0.25))
    assert part == serial
    for info, evs in tls:
        assert info.n_chunks == 1
        check_timeline(info, evs)

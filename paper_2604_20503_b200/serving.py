"""Serving-loop driver over the GPU ServingEngine (the caller of the hot path).

The reference's loop (sim.cpp) is absent from the mount; this follows SPEC.md:541-563 /
SURVEY §3(A): iteration-boundary admission in submit order (B_max = engine max_batch), per
round a speculative length per live request (fixed, or a seeded per-request schedule over
S for bit-exact dynamic-k runs), one ``step()`` (draft -> verify(+EE) -> accept -> commit on
the GPU), finished requests leave after the round.
"""
import time

from . import abi
from .engine import ServingEngine


def run_backlog(eng: ServingEngine, prompts, max_out, k_mode=0, fixed_k=4, k_seed=7,
                gate=None, id_base=0, record=True, max_rounds=0):
    """Submit every prompt, then step until all are done.

    Returns (outputs, records, stats) where records are RoundResult tuples in
    (round, batch order) — the same order oracle/*run_episode logs them.
    """
    for i, (p, m) in enumerate(zip(prompts, max_out)):
        eng.submit(id_base + i, p, m)
    if gate is not None:
        eng.set_gate(gate)
    req_round = {}
    records = []
    stats = dict(rounds=0, drafted=0, submitted=0, accepted=0, committed=0, false_prunes=0,
                 layer_work=0.0, layer_work_full=0.0, finished=0)
    t_first, t_last = {}, {}
    t0 = time.perf_counter()
    while eng.pending_work() > 0:
        if max_rounds and stats["rounds"] >= max_rounds:
            break
        live = eng.live_requests()
        if k_mode == 1:
            ks = [abi.sched_k(k_seed, rid - id_base, req_round.get(rid, 0)) for rid in live]
        else:
            ks = [fixed_k] * len(live)
        eng.set_spec_lengths(live, ks)
        res = eng.step()
        now = time.perf_counter() - t0
        for r in res:
            rid = r.req_id
            req_round[rid] = req_round.get(rid, 0) + 1
            stats["drafted"] += r.drafted
            stats["submitted"] += r.outcome.submitted
            stats["accepted"] += r.outcome.accepted_count
            stats["committed"] += r.committed
            stats["false_prunes"] += r.outcome.false_prune
            stats["layer_work"] += r.outcome.full_layers_run
            stats["layer_work_full"] += eng.params.layers * r.outcome.submitted
            stats["finished"] += r.done
            if r.committed:
                t_first.setdefault(rid, now)
                t_last[rid] = now
            if record:
                t = r.as_tuple()
                records.append((t[0] - id_base,) + t[1:])
        stats["rounds"] += 1
    outs = [eng.committed(id_base + i) for i in range(len(prompts))]
    stats["wall_s"] = time.perf_counter() - t0
    tp = sorted((t_last[i] - t_first[i]) / (len(outs[i - id_base]) - 1)
                for i in t_first if len(outs[i - id_base]) >= 2)
    stats["p50_tpot_ms"] = 1e3 * tp[len(tp) // 2] if tp else 0.0
    return outs, records, stats

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


def synth_trace(mean_rate_per_s=26.0, peak_to_valley=10.0, duration_ms=60000.0, steps=12,
                in_range=(128, 1024), out_range=(64, 256), seed=1):
    """Bursty arrival trace of config 4: sine_segments + synth_workload (workload.cpp:73-114)
    through the product's C ABI. Returns [(arrival_ms, input_len, output_len)]."""
    import ctypes as C

    import numpy as np

    from .engine import lib
    L = lib()
    d, r = np.zeros(steps), np.zeros(steps)
    assert L.faser_sine_segments(C.c_double(mean_rate_per_s), C.c_double(peak_to_valley), C.c_double(duration_ms),
                                 steps, d.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p)) == 0
    n = C.c_int32()
    args = [d.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p), steps, in_range[0], in_range[1],
            out_range[0], out_range[1], C.c_uint64(seed)]
    assert L.faser_synth_workload(*args, None, None, None, 0, C.byref(n)) == 0
    cap = n.value
    a, i, o = np.zeros(max(cap, 1)), np.zeros(max(cap, 1), np.int32), np.zeros(max(cap, 1), np.int32)
    assert L.faser_synth_workload(*args, a.ctypes.data_as(C.c_void_p), i.ctypes.data_as(C.c_void_p),
                                  o.ctypes.data_as(C.c_void_p), cap, C.byref(n)) == 0
    return [(float(a[j]), int(i[j]), int(o[j])) for j in range(cap)]


def run_trace(eng: ServingEngine, trace, vocab, prompt_seed=1, fixed_k=4, id_of=None, clock="device",
              max_steps=0):
    """Replay an arrival trace (the missing sim loop): requests are admitted at
    iteration boundaries once the serving clock has passed their arrival time (B_max =
    engine max_batch, FIFO), one step() per iteration, the clock advances by the step's device
    time (``clock="device"``, CUDA events on the engine stream) or host wall time ("wall"); an
    idle engine jumps to the next arrival. Prompts follow synth_prompt(prompt_seed, trace index).

    Returns per-request records and the MetricsSummary-style aggregates (metrics.hpp:34-66):
    throughput (committed tokens / makespan), p50 TPOT (median over requests of
    (t_last_commit - t_first_commit) / (n_out - 1)), mean TPOT reference-style
    (mean latency_i / n_out_i), p50 / p99 request latency (arrival -> last commit)."""
    import numpy as np

    from .engine import synth_prompt
    ids = id_of or (lambda j: j)
    n = len(trace)
    t_clock = 0.0
    nxt = 0
    arr, first, last, nout = {}, {}, {}, {}
    steps = 0
    t_wall0 = time.perf_counter()
    while nxt < n or eng.pending_work() > 0:
        while nxt < n and trace[nxt][0] <= t_clock:
            a, il, ol = trace[nxt]
            rid = ids(nxt)
            eng.submit(rid, synth_prompt(prompt_seed, nxt, il, vocab), ol)
            arr[rid] = a
            nout[rid] = 0
            nxt += 1
        if eng.pending_work() == 0:
            t_clock = trace[nxt][0]
            continue
        if max_steps and steps >= max_steps:
            break
        live = eng.live_requests()
        eng.set_spec_lengths(live, [fixed_k] * len(live))
        w0 = time.perf_counter()
        res = eng.step()
        dt = eng.last_step_timing()[2] if clock == "device" else (time.perf_counter() - w0) * 1e3
        t_clock += dt
        steps += 1
        for r in res:
            if r.committed:
                first.setdefault(r.req_id, t_clock)
                last[r.req_id] = t_clock
                nout[r.req_id] += r.committed
    done = [rid for rid in arr if nout[rid] > 0]
    tokens = sum(nout.values())
    tpot = sorted((last[r] - first[r]) / (nout[r] - 1) for r in done if nout[r] >= 2)
    lat = sorted(last[r] - arr[r] for r in done)
    t0 = min(arr.values()) if arr else 0.0
    makespan = (max(last.values()) - t0) if last else 0.0
    pct = lambda v, q: float(np.percentile(v, q)) if v else 0.0  # noqa: E731
    return {
        "requests": len(arr), "completed": len(done), "tokens": tokens, "steps": steps,
        "makespan_ms": makespan, "throughput_tok_s": tokens / (makespan / 1e3) if makespan > 0 else 0.0,
        "p50_tpot_ms": pct(tpot, 50), "mean_tpot_ms": float(np.mean([(last[r] - arr[r]) / nout[r] for r in done]))
        if done else 0.0, "p50_latency_ms": pct(lat, 50), "p99_latency_ms": pct(lat, 99),
        "wall_s": time.perf_counter() - t_wall0, "clock": clock,
    }

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


class ModeController:
    """Per-iteration decisions of one AblationMode (config.hpp:16) on top of the
    engine: VSD = fixed k; VSD_AD = AdaptiveDrafter k_i (drafter.cpp:175-220); VSD_AD_EE = + the
    Eq.10 gate (make_gate_plan, exitctl.cpp:70-82, r pinned at 0.5 since should_prune needs
    r in (0,1)); FULL = + the overlap plan (plan_overlap, overlap.cpp:23-42). ``gate_layer`` > 0
    replaces make_gate_plan by a fixed single gated layer; ``chunk`` > 0 forces the overlap chunk."""

    def __init__(self, mode, num_layers, fixed_k=4, models=None, gate_layer=0, chunk=0, profiler=None):
        from . import controller, engine
        self.mode, self.L, self.k, self.models = mode, num_layers, fixed_k, models
        self.gate_layer, self.chunk = gate_layer, chunk
        self.engine = engine
        self.drafter = controller.AdaptiveDrafter(models=models) if mode >= abi.MODE_VSD_AD else None
        # online profiler (profiler.OnlineProfiler): runtime stage samples -> periodic refit of
        # the latency models used below
        self.profiler = profiler
        self.ee_layers = 0
        self.overlap_on = False
        self.r = 1.0  # draft-lane SM share of the plan in force (1.0 = serial, overlap.hpp:14)

    def plan(self, eng, live):
        b = len(live)
        ks = self.drafter.assign_lengths(live, b, self.r) if self.drafter else [self.k] * b
        eng.set_spec_lengths(live, ks)
        if self.mode >= abi.MODE_VSD_AD_EE:
            if self.gate_layer:
                eng.set_gate(abi.GatePlan(self.gate_layer, self.gate_layer + 1, 1.0))
                self.ee_layers = 1
            else:
                # GateEntry.accept_estimate from the AcceptanceBook (drafter.cpp:151-161); the
                # gate's r is the draft share of the overlap plan, 0.5 when serial because
                # should_prune needs r in (0,1) (latmodel.cpp:45)
                a_hat = self.drafter.estimate(live, ks, b, self.r)
                r_gate = self.r if 0.0 < self.r < 1.0 else 0.5
                gp = self.engine.make_gate_plan(abi.ExitPolicy.default(), list(zip(ks, a_hat)),
                                                float(b), r_gate, self.L, self.models)
                eng.set_gate(gp)
                self.ee_layers = max(0, min(gp.stop_layer, self.L) - gp.first_layer)
        self.overlap_on = False
        if self.mode == abi.MODE_FULL:
            if self.chunk:
                self.overlap_on = self.chunk < max(ks)
                eng.set_overlap(self.overlap_on, self.chunk)
            else:
                p = self.engine.plan_overlap(max(ks), len(ks), models=self.models)
                eng.set_overlap(bool(p.enabled), max(p.chunk, 1), p.r)
                self.overlap_on = bool(p.enabled) and p.chunk < max(ks)
        self.r_used = self.r
        self.r = float(eng.plan.overlap.r) if self.overlap_on else 1.0
        return ks

    def observe(self, res, b, step_ms, ks=None, draft_ms=0.0, verify_ms=0.0):
        if self.drafter:
            self.drafter.observe_results(res, b, getattr(self, "r_used", 1.0), max(step_ms, 1e-3))
        if self.profiler is not None and ks is not None:
            serial = not self.overlap_on
            self.profiler.record(b, ks, draft_ms, verify_ms, 1.0 if serial else self.r_used, self.ee_layers)
            m = self.profiler.poll()
            if m is not None:
                self.install_models(m)

    def install_models(self, models):
        """A refreshed latency model: the drafter's GP-LCB objective, the Eq.10 gate and the
        overlap planner use it from the next iteration on."""
        self.models = models
        if self.drafter:
            self.drafter.set_models(models)

    def close(self):
        if self.drafter:
            self.drafter.close()
        if self.profiler is not None:
            self.profiler.close()


MODE_NAMES = {abi.MODE_VSD: "VSD", abi.MODE_VSD_AD: "VSD_AD", abi.MODE_VSD_AD_EE: "VSD_AD_EE", abi.MODE_FULL: "FULL"}


def run_trace(eng: ServingEngine, trace, vocab, prompt_seed=1, fixed_k=4, id_of=None, clock="device",
              max_steps=0, controller=None, num_layers=0, seed=1):
    """Replay an arrival trace (the missing sim loop): requests are admitted at
    iteration boundaries once the serving clock has passed their arrival time (B_max =
    engine max_batch, FIFO), one step() per iteration, the clock advances by the step's device
    time (``clock="device"``, CUDA events on the engine stream) or host wall time ("wall"); an
    idle engine jumps to the next arrival. Prompts follow synth_prompt(prompt_seed, trace index).
    ``controller`` (ModeController) makes the per-iteration mode decisions; default fixed k.

    Returns a dict with the headline numbers and ``summary`` = metrics.MetricsSummary
    (metrics.hpp:34-66): throughput = committed tokens / makespan, p50 TPOT over requests of
    (t_last_commit - t_first_commit) / (n_out - 1), mean TPOT reference-style (mean
    latency_i / n_out_i), request latency arrival -> last commit."""
    import numpy as np

    from . import metrics
    from .engine import synth_prompt
    ids = id_of or (lambda j: j)
    n = len(trace)
    t_clock = 0.0
    nxt = 0
    arr, first, last, nout, fin = {}, {}, {}, {}, {}
    steps = 0
    S = metrics.MetricsSummary(mode=MODE_NAMES.get(eng.cfg.mode, str(eng.cfg.mode)), seed=seed)
    spec_hist, batch_hist = {}, {}
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
        if controller is not None:
            ks = controller.plan(eng, live)
        else:
            ks = [fixed_k] * len(live)
            eng.set_spec_lengths(live, ks)
        w0 = time.perf_counter()
        res = eng.step()
        d_ms, v_ms, s_ms = eng.last_step_timing()
        dt = s_ms if clock == "device" else (time.perf_counter() - w0) * 1e3
        if controller is not None:
            controller.observe(res, len(live), s_ms, ks=ks, draft_ms=d_ms, verify_ms=v_ms)
            S.overlap_iterations += int(controller.overlap_on)
        t_clock += dt
        steps += 1
        S.draft_time_ms += d_ms
        S.verify_time_ms += v_ms
        S.overhead_time_ms += max(0.0, s_ms - d_ms - v_ms)
        batch_hist[len(live)] = batch_hist.get(len(live), 0) + 1
        for k in ks:
            spec_hist[k] = spec_hist.get(k, 0) + 1
        for r in res:
            S.drafted_tokens += r.drafted
            S.submitted_tokens += r.outcome.submitted
            S.accepted_tokens += r.outcome.accepted_count
            S.wasted_draft_tokens += r.drafted - r.outcome.accepted_count
            S.false_prunes += max(0, r.outcome.false_prune)
            S.layer_work += r.outcome.full_layers_run
            S.layer_work_full += num_layers * r.outcome.submitted
            if r.committed:
                first.setdefault(r.req_id, t_clock)
                last[r.req_id] = t_clock
                nout[r.req_id] += r.committed
            if r.done:
                fin[r.req_id] = t_clock
    done = [rid for rid in arr if nout[rid] > 0]
    tokens = sum(nout.values())
    tpot = sorted((last[r] - first[r]) / (nout[r] - 1) for r in done if nout[r] >= 2)
    lat = sorted(last[r] - arr[r] for r in done)
    t0 = min(arr.values()) if arr else 0.0
    makespan = (max(last.values()) - t0) if last else 0.0
    pct = lambda v, q: float(np.percentile(v, q)) if v else 0.0  # noqa: E731
    S.requests, S.finished, S.total_output_tokens = len(arr), len(fin), tokens
    S.makespan_ms = makespan
    S.throughput_tok_s = tokens / (makespan / 1e3) if makespan > 0 else 0.0
    S.mean_request_latency_ms = float(np.mean(lat)) if lat else 0.0
    S.p50_request_latency_ms, S.p99_request_latency_ms = pct(lat, 50), pct(lat, 99)
    S.mean_tpot_ms = float(np.mean([(last[r] - arr[r]) / nout[r] for r in done])) if done else 0.0
    busy = S.draft_time_ms + S.verify_time_ms + S.overhead_time_ms
    S.global_tpot_ms = busy / tokens if tokens else 0.0
    dv = S.draft_time_ms + S.verify_time_ms
    S.verify_share = S.verify_time_ms / dv if dv > 0 else 0.0
    S.acceptance_ratio = S.accepted_tokens / S.submitted_tokens if S.submitted_tokens else 0.0
    S.iterations = steps
    S.spec_length_hist = sorted(spec_hist.items())
    S.batch_size_hist = sorted(batch_hist.items())
    return {
        "requests": len(arr), "completed": len(done), "tokens": tokens, "steps": steps,
        "makespan_ms": makespan, "throughput_tok_s": S.throughput_tok_s,
        "p50_tpot_ms": pct(tpot, 50), "mean_tpot_ms": S.mean_tpot_ms, "p50_latency_ms": S.p50_request_latency_ms,
        "p99_latency_ms": S.p99_request_latency_ms, "wall_s": time.perf_counter() - t_wall0, "clock": clock,
        "summary": S,
    }

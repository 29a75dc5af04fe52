"""bench.py — accepted tokens/s and p50 TPOT of the FASER speculative-decoding data path on B200.

Default workload (BASELINE.json configs[2], "config 3" — the config the metric's batch sweep
1-256 is quoted on): llama-68m-shaped draft / TinyLlama-1.1B-shaped target, random-init bf16
(acceptance-tunable bigram construction), synthetic prompts
(synth_prompt semantics, input U[128,1024], output U[64,256]), continuous batching at B live
requests per GPU (prefill of newly admitted requests happens inside the timed steps), greedy
verification. A "step" is one serving iteration: [admission prefill] -> ragged draft loop ->
verify forward (+ early exit) -> fused accept/commit for every live request.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--batch B] [--k K]
                  [--mode vsd|ad|ee|vsd_ee|full] [--workload cfg3|cfg4|cfg5|toy] [--no-sweep]
                  [--trace SECONDS] [--tp] [--temperature TAU] [--recovery --gate-layer L]
FASER_BENCH_SHARE_GPU=1 (under torchrun): every rank's replica on cuda:0 with a gloo metric
reduction — a functional check of the N > 1 path on a one-GPU box, not a performance number.

Measurement window: before the W warm-up steps every point serves until at least B requests
have finished (<= FILL_CAP untimed steps), so the K timed steps see the steady-state mix of
admissions (prefill), decoding requests and completions instead of the first batch's
admission burst; the number does not depend on K beyond sampling noise.
batch_sweep: the same measurement at B in SWEEP (1, 8, 32, 128, 256), each with its own
roofline under the right bound (tensor when B*k rows exceed the ridge, HBM below).

value      : committed tokens / device time of the K steps (CUDA events on the engine stream,
             max over ranks), prompts submitted to the engine before the timed region.
e2e        : the same metric through the C ABI with HOST buffers: prompts submitted from host
             memory inside the timed region, per-step H2D of the step plan + admissions and D2H
             of the round results, wall clock.
reference  : `--impl reference` runs the reference semantics on the host CPU: for cfg3 the
             fp32 oracle port (oracle/lmsd.py — the reference has no transformer path) on the
             SAME backlog (prompts from the reference's own compiled synth_prompt, whole request
             lifetimes incl. prefill) and the same `config`; for the toy workload the reference's
             own compiled engine (oracle/_ref). It never loads the product library.
Multi-GPU  : requests are sharded across ranks (independent replicas, no collective on the
             data path); value = all ranks' tokens / max-over-ranks device time.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2604_20503_b200 import abi  # noqa: E402

METRIC = "accepted tokens/sec (committed output tokens per second)"
WORKLOAD_NAMES = {
    "cfg3": "config 3: llama-68m-shape draft / TinyLlama-1.1B-shape target",
    "cfg4": "config 4: Llama-3.2-1B-shape draft / Llama-3.1-8B-shape target",
    "cfg5": "config 5: Llama-3.2-1B-shape draft / Llama-3.1-70B-shape target",
    "tiny": "tiny test pair", "tp_tiny": "tiny TP test pair",
}
UNIT = "tokens/s"


# ------------------------------------------------------------------ shared helpers
class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.max_mhz = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                self.samples.append(float(out[0]))
                self.max_mhz = float(out[1])
                for nm, v in zip(names, out[2:]):
                    if v.strip().lower() == "active":
                        self.reasons.add(nm)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def lens(seed, n, in_range, out_range):
    """synth_workload's `lens` substream (workload.cpp:77,89-90): input then output length per
    record, SplitMixStream(substream(seed, 'lens')), next_int with modulo (rng.hpp:67-70)."""
    M = (1 << 64) - 1
    G = 0x9E3779B97F4A7C15
    state = abi.mix64(abi.mix64(seed ^ abi.mix64(0x6C656E73)) & M)
    ins, outs = [], []
    for _ in range(n):
        state = (state + G) & M
        ins.append(in_range[0] + abi.mix64(state) % (in_range[1] - in_range[0] + 1))
        state = (state + G) & M
        outs.append(out_range[0] + abi.mix64(state) % (out_range[1] - out_range[0] + 1))
    return ins, outs


def prompts_for(base, n, vocab, in_range, out_range, seed=1):
    """synth_prompt(seed, idx, len, V) (workload.cpp:116-122) via the product's C ABI."""
    import ctypes as C

    import numpy as np

    from paper_2604_20503_b200 import engine
    L = engine.lib()
    inl, outl = lens(seed, base + n, in_range, out_range)
    out = []
    for i in range(base, base + n):
        buf = np.zeros(inl[i], np.int32)
        assert L.faser_synth_prompt(C.c_uint64(seed), i, inl[i], vocab, buf.ctypes.data_as(C.c_void_p)) == 0
        out.append(buf.tolist())
    return out, outl[base:base + n]


def shard_base(rank, n_req):
    """Request-sharded replicas: rank r owns requests [r*n_req, (r+1)*n_req) of the workload
    (synth_prompt is indexed, so the shards are disjoint and their union is the 1-GPU run)."""
    return rank * n_req


def shard_trace(trace, rank, world):
    """Request-sharded trace replay: rank r owns trace indices r, r+N, ... (arrival order kept);
    returns [(trace index, record)]."""
    return [(j, trace[j]) for j in range(rank, len(trace), world)]


def llama_trace(args, rank, world, local_rank):
    """Bursty arrival-trace replay (config 4, BASELINE.json configs[3]): sine_segments(mean
    26 req/s, peak/valley 10, 12 steps) over --trace seconds (workload.cpp:73-114), requests
    sharded over ranks, per-rank serving clock = device time of its steps; whole-job tokens/s =
    sum of tokens / max over ranks of the makespan, p50 TPOT over the union of requests."""
    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(DIST_BACKEND)
    from paper_2604_20503_b200 import serving
    desc = llama_desc(args.workload)
    V = desc.target.vocab
    trace = serving.synth_trace(mean_rate_per_s=args.trace_rate, peak_to_valley=10.0,
                                duration_ms=args.trace * 1e3, steps=12, in_range=IN_RANGE,
                                out_range=OUT_RANGE, seed=1)
    mine = shard_trace(trace, rank, world)
    eng = make_engine(desc, args, local_rank)
    # warm-up on a few private requests (ids past the trace), not timed
    for i in range(min(4, args.batch)):
        eng.submit(10 ** 9 + i, [1 + i, 2, 3, 4, 5], 8)
    while eng.pending_work() > 0:
        eng.step()
    ids = [j for j, _ in mine]
    m = serving.run_trace(eng, [rec for _, rec in mine], V, prompt_seed=1, fixed_k=args.k,
                          id_of=lambda q: ids[q])
    eng.close()
    vals = torch.tensor([m["makespan_ms"], float(m["tokens"]), m["p50_tpot_ms"], float(m["requests"])],
                        dtype=torch.float64, device="cuda")
    if dist is not None:
        g = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(g, vals)
        allv = torch.stack(g).cpu()
    else:
        allv = vals.cpu()[None]
    if rank == 0:
        mk = float(allv[:, 0].max())
        tok = float(allv[:, 1].sum())
        print(json.dumps({
            "metric": METRIC, "value": tok / (mk / 1e3), "unit": UNIT, "n_gpus": world, "steps": m["steps"],
            "warmup": 1, "ms_per_step": mk / max(1, m["steps"]), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic bursty trace (sine_segments + synth_workload), random-init weights",
            "p50_tpot_ms_rank0": m["p50_tpot_ms"], "p50_tpot_ms_ranks": allv[:, 2].tolist(),
            "config": {"workload": f"{args.workload}: bursty trace replay, mean {args.trace_rate} req/s, peak/valley 10, "
                       f"{args.trace} s, 12 segments, k={args.k}, B_max={args.batch}/GPU",
                       "global_batch": args.batch * world, "requests": len(trace),
                       "parallelism": f"replicas x{world} (request-sharded trace)", "clock": "device time of the steps"},
            "trace_rank0": {k: v for k, v in m.items() if k != "summary"},
            "summary_rank0": m["summary"].as_json()}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# process-group backend of the N > 1 metric reduction (the data path has no collective)
DIST_BACKEND = "gloo" if os.environ.get("FASER_BENCH_SHARE_GPU") == "1" else "nccl"


def aggregate(stats, dist):
    """Whole-job numbers: device time and e2e wall time are the MAX over ranks, tokens the SUM.
    stats = [dev_ms, tokens, e2e_s, e2e_tokens] (float64 tensor on this rank's device)."""
    if dist is None:
        return [float(x) for x in stats.tolist()]
    mx = stats.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = stats.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return [mx[0].item(), sm[1].item(), mx[2].item(), sm[3].item()]


def p50_tpot_ms(first, last):
    tp = [(last[r][0] - first[r]) / (last[r][1] - 1) for r in last if last[r][1] >= 2]
    return 1e3 * statistics.median(tp) if tp else None


def mean_tpot_ms(first, last):
    """metrics.hpp:45's mean over requests, of each request's per-token time inside the window"""
    tp = [(last[r][0] - first[r]) / (last[r][1] - 1) for r in last if last[r][1] >= 2]
    return 1e3 * statistics.fmean(tp) if tp else None


# ------------------------------------------------------------------ Llama workload (config 3)
IN_RANGE, OUT_RANGE = (128, 1024), (64, 256)


def llama_desc(name):
    from paper_2604_20503_b200 import llama
    return llama.PRESETS[name]()


def make_engine(desc, args, local_rank, batch=None, **tp):
    from paper_2604_20503_b200 import engine
    mode = {"vsd": abi.MODE_VSD, "ad": abi.MODE_VSD_AD, "ee": abi.MODE_VSD_AD_EE,
            "ov": abi.MODE_FULL, "full": abi.MODE_FULL, "vsd_ee": abi.MODE_VSD_AD_EE}[args.mode]
    eng = engine.ServingEngine(desc=desc, max_batch=batch or args.batch, max_seq_len=IN_RANGE[1] + OUT_RANGE[1] + 8,
                               mode=mode, default_spec_length=args.k, max_spec_length=16,
                               prefill_rows=8192, device=local_rank,
                               prefill_lane=0 if (tp or args.no_prefill_lane) else 1,
                               exempt_rule=2 if getattr(args, "recovery", False) else 1, **tp)
    if getattr(args, "temperature", 0.0) > 0.0:  # coupled Gumbel-max sampling acceptance
        eng.set_sampling(args.temperature, 1)
    return eng


def tp_bootstrap(dist, rank, make_uid):
    """NCCL TP group bootstrap: rank 0 makes the 128-byte ncclUniqueId, every rank receives it
    through the launcher's process group (torch.distributed is plumbing only)."""
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def llama_tp(args, rank, world, local_rank):
    """Config 5 (BASELINE.json configs[4]): TP=world verification of the 70B-shaped target, one
    process per GPU, NCCL all-reduce after O / down and all-gathered vocab-parallel argmax. All
    ranks serve the SAME requests (tensor parallel, not request-sharded); tokens are counted once,
    time = max over ranks of the device time."""
    import torch
    torch.cuda.set_device(local_rank)
    import torch.distributed as dist
    dist.init_process_group("nccl" if world > 1 else "gloo", init_method=None if world > 1 else "tcp://127.0.0.1:29533",
                            rank=rank, world_size=world)
    from paper_2604_20503_b200 import engine
    uid = tp_bootstrap(dist, rank, engine.TpGroup.nccl_unique_id)
    group = engine.TpGroup.nccl(uid, world, rank, local_rank)
    desc = llama_desc(args.workload)
    V = desc.target.vocab
    B = args.batch
    n_req = B * (args.steps + args.warmup) // 40 + 2 * B
    prompts, outl = prompts_for(0, n_req, V, IN_RANGE, OUT_RANGE)
    eng = make_engine(desc, args, local_rank, tp_size=world, tp_rank=rank, tp_group=group)
    for i, (p, m) in enumerate(zip(prompts, outl)):
        eng.submit(i, p, m)
    for _ in range(args.warmup):
        eng.step()
    dist.barrier()
    torch.cuda.synchronize()
    dev_ms, tokens, first, last, clock = 0.0, 0, {}, {}, 0.0
    ph = [0.0, 0.0]  # draft (+ admission) / verify + accept device ms over the timed steps
    for _ in range(args.steps):
        res = eng.step()
        tm = eng.last_step_timing()
        dt = tm[2]
        ph[0] += tm[0]
        ph[1] += tm[1]
        dev_ms += dt
        clock += dt
        for r in res:
            tokens += r.committed
            if r.committed:
                first.setdefault(r.req_id, clock)
                last[r.req_id] = clock
    torch.cuda.synchronize()
    t = torch.tensor([dev_ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tp50 = sorted((last[i] - first[i]) / max(1, len(eng.committed(i)) - 1) for i in first if len(eng.committed(i)) > 1)
    if rank == 0:
        ms = float(t[0])
        print(json.dumps({
            "metric": METRIC, "value": tokens / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic prompts (synth_prompt), random-init weights",
            "p50_tpot_ms": tp50[len(tp50) // 2] if tp50 else 0.0,
            "config": {"workload": f"{args.workload}: TP={world} verification (NCCL all-reduce after O/down, "
                       f"vocab-parallel argmax), replicated draft, B={B}, k={args.k}", "global_batch": B,
                       "parallelism": f"tp{world}"},
            "device_ms_per_step": {"draft": ph[0] / args.steps, "verify_accept": ph[1] / args.steps},
            # per rank: each streams 1/world of the target's weights (and KV heads) per verify
            "verify_forward_roofline": tp_rank_roofline(llama_roofline(desc, B, args.k, ph[1] / args.steps), world)}),
              flush=True)
    eng.close()
    group.close()
    dist.destroy_process_group()


def gate_plan(desc, args):
    """Fixed gate (--gate-layer l: gate exactly layer l) or None = per-step make_gate_plan
    (exitctl.cpp:70-82) on the B200-fitted latency models."""
    if args.mode not in ("ee", "vsd_ee") or not args.gate_layer:
        return None
    return abi.GatePlan(args.gate_layer, args.gate_layer + 1, 1.0)


def step_plan_hook(desc, args, models, book=None):
    """Per-step controller decisions that need the batch: the early-exit gate (make_gate_plan
    with GateEntry.accept_estimate from the AcceptanceBook `book` (drafter.cpp:151-161), r pinned
    at 0.5 as should_prune requires r in (0,1)) and the overlap plan (plan_overlap)."""
    from paper_2604_20503_b200 import engine
    L = desc.target.layers

    def hook(eng, live, ks):
        if args.mode in ("ee", "vsd_ee") and not args.gate_layer:
            a_hat = book.estimate(live, ks, len(live), 1.0) if book is not None else [0.6] * len(ks)
            eng.set_gate(engine.make_gate_plan(abi.ExitPolicy.default(), list(zip(ks, a_hat)),
                                               float(len(ks)), 0.5, L, models))
        if args.mode in ("ov", "full"):
            if args.chunk:
                eng.set_overlap(True, args.chunk)
            else:
                p = engine.plan_overlap(max(ks), len(ks), models=models)
                eng.set_overlap(bool(p.enabled), max(p.chunk, 1), p.r)
    return hook


def run_llama_steps(eng, n_steps, clock, state, feeder=None, gate=None, drafter=None, chunk=0, hook=None,
                    book=None):
    """n_steps serving iterations; per-request first/last commit times on `clock`. With a
    drafter (AdaptiveDrafter) the per-request k_i come from assign_lengths before each step and
    the round is fed back with observe_round after it (the reference loop).
    Returns the committed tokens; state["steps"] counts the steps actually executed and
    state["finished"] the requests that completed."""
    tokens = 0
    prof = HOST_PROF if os.environ.get("BENCH_HOST_PROF") == "1" else None
    for _ in range(n_steps):
        t_a = time.perf_counter()
        if feeder is not None:
            feeder()
        live = eng.live_requests()
        if not live:
            break
        ks = None
        if drafter is not None:
            ks = drafter.assign_lengths(live, len(live), drafter_r(eng))
            eng.set_spec_lengths(live, ks)
        if gate is not None:
            eng.set_gate(gate)
        if hook is not None:
            hook(eng, live, ks or [eng.cfg.default_spec_length] * len(live))
        t_b = time.perf_counter()
        res = eng.step()
        t_c = time.perf_counter()
        state["steps"] = state.get("steps", 0) + 1
        for r in res:
            state["acc"] = state.get("acc", 0) + r.outcome.accepted_count
            state["sub"] = state.get("sub", 0) + r.outcome.submitted
            state["flr"] = state.get("flr", 0.0) + r.outcome.full_layers_run
            state["finished"] = state.get("finished", 0) + (1 if r.done else 0)
        for obs in {id(x): x for x in (drafter, book) if x is not None}.values():
            obs.observe_results(res, len(live), drafter_r(eng), max(eng.last_step_timing()[2], 1e-3))
        now = clock()
        for r in res:
            if r.committed:
                tokens += r.committed
                state["first"].setdefault(r.req_id, now)
                n0 = state["last"].get(r.req_id, (0, 0))[1]
                state["last"][r.req_id] = (now, n0 + r.committed)
        if prof is not None:
            t_d = time.perf_counter()
            prof["pre_ms"] += 1e3 * (t_b - t_a)
            prof["step_ms"] += 1e3 * (t_c - t_b)
            prof["post_ms"] += 1e3 * (t_d - t_c)
            prof["steps"] += 1
    return tokens


HOST_PROF = {"pre_ms": 0.0, "step_ms": 0.0, "post_ms": 0.0, "steps": 0}  # BENCH_HOST_PROF=1


def drafter_r(eng):
    """SM share the AdaptiveDrafter sees (assign_lengths(b, r), drafter.hpp:105-107): the draft
    lane's share of the overlap plan in force, 1.0 for serial execution (overlap.hpp:14)."""
    ov = getattr(eng, "overlap_state", None)
    if ov and ov[0]:
        return float(ov[2])
    return 1.0


# ---------------------------------------------------------------- backlog + steady state
REQS_PER_RANK = 1 << 20  # index space per rank: request-sharded replicas own disjoint blocks
FILL_CAP = 400           # max untimed steps spent bringing the server to steady state
SWEEP = (1, 8, 32, 128, 256)


class Backlog:
    """The workload's request stream for one rank: request i = (synth_prompt(1, base+i, len_i,
    V), max_out_i) with lengths from synth_workload's `lens` substream (workload.cpp:77,89-122),
    generated lazily. `synth` is the prompt generator (the product's C ABI for our arm, the
    reference's own compiled workload.cpp for the reference arm)."""

    def __init__(self, base, vocab, synth, n_lens=4096):
        self.base, self.vocab, self.synth = base, vocab, synth
        self.ins, self.outs = lens(1, base + n_lens, IN_RANGE, OUT_RANGE)
        self.next = 0

    def take(self):
        i = self.base + self.next
        if i >= len(self.ins):
            self.ins, self.outs = lens(1, 2 * len(self.ins), IN_RANGE, OUT_RANGE)
        self.next += 1
        return i, self.synth(i, self.ins[i]), self.outs[i]


def product_synth(vocab):
    import ctypes as C

    import numpy as np

    from paper_2604_20503_b200 import engine
    L = engine.lib()

    def synth(i, n):
        buf = np.zeros(n, np.int32)
        assert L.faser_synth_prompt(C.c_uint64(1), i, n, vocab, buf.ctypes.data_as(C.c_void_p)) == 0
        return buf.tolist()
    return synth


def reference_synth(vocab):
    """synth_prompt from the reference's own workload.cpp compiled in place (oracle/_ref); the
    restated C oracle when the reference build is absent. Never loads the product library."""
    from oracle import pyoracle as po
    o = po.ref() if os.path.exists(po.REF_SO) else po.restated()
    return (lambda i, n: list(o.synth_prompt(1, i, n, vocab))), ("reference" if o is not po.restated() else "port")


def llama_config(args, world, B):
    """The `config` object both arms print (identical by construction)."""
    return {"workload": f"{WORKLOAD_NAMES.get(args.workload, args.workload)}, continuous batching "
                        f"B={B}/GPU, k={args.k}, mode={args.mode}, steady state (>= one request "
                        f"lifetime served before warm-up)",
            **({"temperature": args.temperature, "acceptance_rule": "coupled Gumbel-max sampling"}
               if getattr(args, "temperature", 0.0) > 0.0 else {}),
            "global_batch": B * world, "seq_len": f"in U{list(IN_RANGE)} out U{list(OUT_RANGE)}",
            "parallelism": f"replicas x{world} (request-sharded)",
            "l2": "target weights per verify >> 126 MB L2 (inputs larger than L2)"}


def serve_point(args, desc, B, rank, world, local_rank, dist, want_e2e, want_kstats):
    """One batch size: [fill to steady state] -> W warm-up steps -> K timed steps (device
    time, CUDA events on the engine stream) -> kernel-class timing steps; optionally the e2e
    leg on a fresh engine (host prompts submitted inside the timed region, wall clock)."""
    import torch
    from paper_2604_20503_b200 import llama as _llama
    V = desc.target.vocab
    gate = gate_plan(desc, args)
    models = _llama.fitted_latency_model()
    synth = product_synth(V)

    def new_drafter():
        if args.mode in ("vsd", "ov", "vsd_ee"):
            return None
        from paper_2604_20503_b200 import controller
        return controller.AdaptiveDrafter(models=models)

    def new_book():
        """AcceptanceBook for the early-exit gate when k is fixed (no AdaptiveDrafter choosing k)."""
        if args.mode not in ("vsd_ee",):
            return None
        from paper_2604_20503_b200 import controller
        return controller.AdaptiveDrafter(models=models)

    def sync_all():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def session(eng, counting=False):
        bl = Backlog(shard_base(rank, REQS_PER_RANK), V, synth)
        io = {"sub": 0, "h2d": 0, "d2h": 0, "counting": False}

        def feeder():
            if io["counting"]:
                a, b = eng.last_step_bytes()
                io["h2d"] += a
                io["d2h"] += b
            while eng.pending_work() < B + 2:
                i, p, m = bl.take()
                eng.submit(i, p, m)
                if io["counting"]:
                    io["sub"] += 4 * len(p)
        return feeder, io

    def fill(eng, feeder, drafter, clock):
        st = {"first": {}, "last": {}}
        n = 0
        while n < FILL_CAP and st.get("finished", 0) < B:
            run_llama_steps(eng, 1, clock, st, feeder, gate=gate, drafter=drafter, hook=hook, book=book)
            n += 1
        return n

    # ------------------------------------------------------------ value (device-timed)
    eng = make_engine(desc, args, local_rank, batch=B)
    feeder, _ = session(eng)
    dev_clock = [0.0]

    def clock():
        dev_clock[0] += eng.last_step_timing()[2] / 1e3
        return dev_clock[0]

    drafter = new_drafter()
    book = drafter or new_book()
    hook = step_plan_hook(desc, args, models, book)
    fill_steps = fill(eng, feeder, drafter, clock)
    run_llama_steps(eng, args.warmup, clock, {"first": {}, "last": {}}, feeder, gate=gate, drafter=drafter,
                    hook=hook, book=book)
    stream = torch.cuda.ExternalStream(eng.stream_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = {"first": {}, "last": {}}
    dev_clock[0] = 0.0
    launches0 = eng.kernel_launches()
    acc_ms = {"prefill": 0.0, "draft": 0.0, "verify": 0.0}

    def clock_acc():
        d, v, _ = eng.last_step_timing()
        pf = eng.last_step_prefill_ms()
        acc_ms["prefill"] += pf
        acc_ms["draft"] += d - pf
        acc_ms["verify"] += v
        return clock()

    sync_all()
    with Clocks(local_rank) as clk:
        ev0.record(stream)
        t0 = time.perf_counter()
        tokens = run_llama_steps(eng, args.steps, clock_acc, st, feeder, gate=gate, drafter=drafter, hook=hook, book=book)
        eng.join_lanes()  # the last admissions' prefill (side lane) inside the timed region
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    launches = eng.kernel_launches() - launches0
    dev_ms = ev0.elapsed_time(ev1)
    nsteps = max(st.get("steps", 0), 1)
    out = {"B": B, "dev_ms": dev_ms, "tokens": tokens, "steps_run": st.get("steps", 0), "fill_steps": fill_steps,
           "p50_tpot_ms": p50_tpot_ms(st["first"], st["last"]), "mean_tpot_ms": mean_tpot_ms(st["first"], st["last"]),
           "accepted_draft": st.get("acc", 0), "launches": launches, "clocks": clk.summary(),
           "wall_s": wall, "draft_ms": acc_ms["draft"] / nsteps, "verify_ms": acc_ms["verify"] / nsteps,
           "prefill_ms": acc_ms["prefill"] / nsteps,
           "acceptance": st.get("acc", 0) / max(st.get("sub", 1), 1),
           "layer_work": st.get("flr", 0.0) / max(st.get("sub", 1), 1)}
    if want_kstats:
        # per-kernel-class CUDA-event timing over steps that immediately follow the timed region
        # (event records between launches would perturb the PDL overlap being timed); the
        # prefill lane is off for them, so each class is timed without a co-running prefill
        if not args.no_prefill_lane:
            eng.set_prefill_lane(False)
        eng.set_kernel_timing(True)
        run_llama_steps(eng, max(args.steps // 2, 3), clock, {"first": {}, "last": {}}, feeder, gate=gate,
                        drafter=drafter, hook=hook, book=book)
        out["kstats"] = eng.kernel_stats()
        eng.set_kernel_timing(False)
        # in-stream class costs: verify time of interleaved steps with all kernels, without the
        # projection GEMMs (skip mask 30) and without attention (mask 1); no events between
        # launches, so PDL overlap is intact. The skipping steps compute garbage, which is why
        # this runs last, right before the engine is closed.
        vt = {-1: [], 30: [], 1: []}
        for i in range(18):
            if not eng.live_requests():
                break
            m = (-1, 30, 1)[i % 3]
            eng.debug_set_skip_mask(m)
            feeder()
            eng.step()
            vt[m].append(eng.last_step_timing()[1])
        eng.debug_set_skip_mask(-1)
        out["instream_verify_ms"] = {str(k): sum(v) / len(v) for k, v in vt.items() if v}
    eng.close()
    if not want_e2e:
        return out

    # ------------------------------------------------------------ e2e (host buffers, wall clock)
    eng = make_engine(desc, args, local_rank, batch=B)
    feeder, io = session(eng)
    drafter2 = new_drafter()
    book = drafter2 or new_book()
    hook = step_plan_hook(desc, args, models, book)
    fill(eng, feeder, drafter2, time.perf_counter)
    run_llama_steps(eng, args.warmup, time.perf_counter, {"first": {}, "last": {}}, feeder, gate=gate,
                    drafter=drafter2, hook=hook, book=book)
    sync_all()
    io["counting"] = True
    eng.last_step_bytes()
    st2 = {"first": {}, "last": {}}
    t0 = time.perf_counter()
    tokens2 = run_llama_steps(eng, args.steps, time.perf_counter, st2, feeder, gate=gate, drafter=drafter2,
                              hook=hook)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    a, b = eng.last_step_bytes()
    io["h2d"] += a
    io["d2h"] += b
    eng.close()
    n2 = max(st2.get("steps", 0), 1)
    out["e2e"] = {"s": e2e_s, "tokens": tokens2, "p50_tpot_ms": p50_tpot_ms(st2["first"], st2["last"]),
                  "h2d_bytes_per_step": int((io["h2d"] + io["sub"]) / n2), "d2h_bytes_per_step": int(io["d2h"] / n2)}
    return out


def llama_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(DIST_BACKEND)
    desc = llama_desc(args.workload)
    B = args.batch
    head = serve_point(args, desc, B, rank, world, local_rank, dist, want_e2e=True, want_kstats=True)
    points = [head]
    if not args.no_sweep:
        for b in SWEEP:
            if b != B:
                points.append(serve_point(args, desc, b, rank, world, local_rank, dist, want_e2e=False,
                                          want_kstats=True))
    # whole-job reduction per point: device time / wall = max over ranks, tokens = sum
    agg = []
    for p in points:
        e = p.get("e2e", {"s": 0.0, "tokens": 0})
        stats = torch.tensor([p["dev_ms"], float(p["tokens"]), e["s"], float(e["tokens"])], dtype=torch.float64,
                             device="cuda")
        agg.append(aggregate(stats, dist))
    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    dev_ms, tokens, e2e_s, tokens2 = agg[0]
    line = {
        "metric": METRIC, "value": tokens / (dev_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "steps_executed": head["steps_run"],
        "ms_per_step": dev_ms / max(head["steps_run"], 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts (synth_prompt), random-init weights",
        "p50_tpot_ms": head["p50_tpot_ms"],
        "mean_tpot_ms": head["mean_tpot_ms"],
        # accepted drafted tokens per second (metrics.hpp:53; committed = these + recovery tokens), rank 0
        "accepted_draft_tokens_per_s": head["accepted_draft"] / (head["dev_ms"] / 1e3),
        "config": llama_config(args, world, B),
        "e2e": {"value": tokens2 / e2e_s, "unit": UNIT, "p50_tpot_ms": head["e2e"]["p50_tpot_ms"],
                "h2d_bytes_per_step": head["e2e"]["h2d_bytes_per_step"],
                "d2h_bytes_per_step": head["e2e"]["d2h_bytes_per_step"]},
        "gpu_launches": int(head["launches"]),
        "clocks": head["clocks"],
        "device_ms_per_step": {"admit_prefill": head["prefill_ms"], "draft": head["draft_ms"],
                               "verify_accept": head["verify_ms"]},
        "acceptance": head["acceptance"],
        "layer_work_per_drafted_token": head["layer_work"],
        "fill_steps": head["fill_steps"],
        "wall_s_timed": head["wall_s"],
    }
    line["roofline"], line["kernels"] = kernel_roofline(head["kstats"], B * args.k)
    inst = instream_roofline(head, desc, line["kernels"])
    if inst and line["roofline"]:
        line["roofline"]["instream"] = inst
    line["verify_forward_roofline"] = llama_roofline(desc, B, args.k, head["verify_ms"])
    sweep = []
    for p, (d_ms, tok, _, _) in zip(points, agg):
        roof, _ = kernel_roofline(p["kstats"], p["B"] * args.k)
        sweep.append({"batch": p["B"], "global_batch": p["B"] * world, "value": tok / (d_ms / 1e3),
                      "p50_tpot_ms": p["p50_tpot_ms"], "ms_per_step": d_ms / max(p["steps_run"], 1),
                      "steps_executed": p["steps_run"], "fill_steps": p["fill_steps"],
                      "acceptance": p["acceptance"], "clocks_sm_mhz": p["clocks"]["sm_mhz"],
                      "roofline": roof})
    line["batch_sweep"] = sorted(sweep, key=lambda x: x["batch"])
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = llama_cpu_sample(desc, args, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)
    if os.environ.get("BENCH_HOST_PROF") == "1":
        print("host per step (all run_llama_steps calls): " + json.dumps({k: (v / max(HOST_PROF["steps"], 1) if k != "steps" else v) for k, v in HOST_PROF.items()}), file=sys.stderr)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def instream_roofline(head, desc, kernels):
    """The verify GEMM and attention classes' cost inside the step stream (PDL overlap intact):
    verify time with every kernel minus verify time with the class skipped (interleaved steps,
    FASER_SKIP masks through faser_debug_set_skip_mask), per launch, against the same
    algorithmic bytes per launch as the event-timed classes."""
    v = head.get("instream_verify_ms") or {}
    if "-1" not in v or "30" not in v or not kernels:
        return None
    pk, src = peaks()
    L = desc.target.layers
    res = {"method": "verify ms with all kernels minus with the class skipped, interleaved steps, / launches",
           "verify_ms": v["-1"]}
    for cls, mask, per_layer in (("verify_gemm", "30", 4), ("verify_attention", "1", 1)):
        if cls not in kernels or mask not in v:
            continue
        us = 1e3 * (v["-1"] - v[mask]) / (L * per_layer)
        if us <= 0:
            continue
        gbs = kernels[cls]["bytes_per_launch"] / (us * 1e-6) / 1e9
        res[cls] = {"avg_launch_us": us, "achieved_GBs": gbs, "frac_hbm": gbs / pk["hbm_gbs"]}
        if kernels[cls].get("flops_per_launch"):
            tfs = kernels[cls]["flops_per_launch"] / (us * 1e-6) / 1e12
            peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
            res[cls].update({"achieved_TFs": tfs, "frac_tensor": tfs / peak})
    return res


def kernel_roofline(kstats, rows):
    """roofline object for the dominant kernel class (largest device time). `rows` = verify rows
    per step (B*k): below the ridge (peak flops / peak bytes, ~216 rows for bf16 on B200) the
    GEMM classes are HBM-bound (achieved = algorithmic bytes per launch / average launch time vs
    the measured copy bandwidth), above it tensor-bound (algorithmic flops per launch / time vs
    the sustained bf16 matmul rate). Attention classes are always HBM-bound."""
    pk, src = peaks()
    ridge = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * 1e12 / (pk["hbm_gbs"] * 1e9)
    table = {}
    for name, v in kstats.items():
        if v["launches"]:
            gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9
            tfs = v.get("flops", 0.0) / (v["ms"] * 1e-3) / 1e12
            table[name] = {"avg_us": 1e3 * v["ms"] / v["launches"], "launches": v["launches"],
                           "bytes_per_launch": v["bytes"] / v["launches"], "achieved_GBs": gbs,
                           "frac_hbm": gbs / pk["hbm_gbs"], "total_ms": v["ms"],
                           "flops_per_launch": v.get("flops", 0.0) / v["launches"], "achieved_TFs": tfs}
    if not table:
        return None, table
    top = max(table, key=lambda n: table[n]["total_ms"])
    t = table[top]
    tensor = "gemm" in top or "lm_head" in top
    tensor = tensor and rows >= ridge and t["flops_per_launch"] > 0
    traffic = None  # dram__bytes_read.sum + dram__bytes_write.sum per launch, committed ncu capture
    for fn in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                traffic = json.load(f)["classes"][top]["traffic_bytes_per_launch"]
            break
        except Exception:
            pass
    share = t["total_ms"] / sum(x["total_ms"] for x in table.values())
    if tensor:
        peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        roof = {"bound": "tensor", "achieved": t["achieved_TFs"], "peak": peak, "unit": "TFLOP/s",
                "frac": t["achieved_TFs"] / peak, "traffic": traffic, "peak_source": src + " bf16_tflops_sustained"}
    else:
        roof = {"bound": "hbm", "achieved": t["achieved_GBs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": t["achieved_GBs"] / pk["hbm_gbs"], "traffic": traffic, "peak_source": src + " hbm_gbs"}
    roof.update({"kernel": top, "avg_launch_us": t["avg_us"], "bytes_per_launch": t["bytes_per_launch"],
                 "flops_per_launch": t["flops_per_launch"], "rows": rows, "ridge_rows": ridge,
                 "share_of_timed_kernels": share})
    return roof, table


def llama_roofline(desc, B, k, verify_ms):
    """Dominant path = the verify forward (target weights streamed once per step). Algorithmic
    bytes per verify = 2 * target params (bf16) + KV read (sum ctx * KV bytes/token), SURVEY 8(d)."""
    pk, src = peaks()
    t = desc.target
    d, L, F, V = t.d_model, t.layers, t.ffn, t.vocab
    qkv = (t.n_heads + 2 * t.n_kv_heads) * t.head_dim
    params = L * (qkv * d + d * t.n_heads * t.head_dim + 3 * d * F) + V * d  # + LM head
    kv_tok = 2 * L * t.n_kv_heads * t.head_dim * 2
    mean_ctx = (IN_RANGE[0] + IN_RANGE[1]) / 2 + (OUT_RANGE[0] + OUT_RANGE[1]) / 4
    bytes_ = 2 * params + B * mean_ctx * kv_tok
    achieved = bytes_ / (verify_ms * 1e-3) / 1e9 if verify_ms else 0.0
    return {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": None, "peak_source": src,
            "kernel": "target verify forward (tcgen05 GEMMs + paged attention + accept), per step",
            "algorithmic_bytes": bytes_, "rows_per_verify": B * k}


def tp_rank_roofline(roof, world):
    """A TP rank streams 1/world of the verify's algorithmic bytes in the same time."""
    if world <= 1:
        return roof
    r = dict(roof)
    r["algorithmic_bytes"] = roof["algorithmic_bytes"] / world
    r["achieved"] = roof["achieved"] / world
    r["frac"] = roof["frac"] / world
    r["note"] = f"per rank: 1/{world} of the target's weights and KV"
    return r


def llama_cpu_sample(desc, args, budget_s=20.0):
    """The reference's speculative-decoding semantics on the host cores over the fp32 oracle
    models (oracle/lmsd.py: draft_tokens / full_verify / commit of sdcore.cpp:45-197 with the
    transformer pair in place of LayeredToyLM; the reference has no transformer). SAME workload
    as the GPU arm: requests of the same backlog in order (prompts from the reference's own
    compiled synth_prompt, lengths from the `lens` substream), k fixed. The reference engine's
    API is per request (SpeculativeEngine methods take one Request, sdcore.hpp:81-116), so a
    batch of B live requests costs the sum of their per-request rounds and throughput does not
    depend on B: the bounded sample is whole request lifetimes (admission prefill + every round
    to completion), run one after another until `budget_s` is spent. Never loads the product
    library."""
    from oracle import lmsd
    threads = os.cpu_count() or 1
    V = desc.target.vocab
    synth, kind = reference_synth(V)
    bl = Backlog(0, V, synth, n_lens=64)
    sd = lmsd.OracleSD(desc, threads)
    tok = rounds = nreq = 0
    spent = 0.0
    prefill_tok = 0
    while spent < budget_s and nreq < 64:
        t0 = time.perf_counter()
        i, p, m = bl.take()
        sd.submit(i, p, m)
        while not sd.reqs[i].done:
            tok += sd.round(i, args.k)[3]
            rounds += 1
        spent += time.perf_counter() - t0
        sd.release(i)
        nreq += 1
        prefill_tok += len(p)
    sd.close()
    return {"value": tok / spent, "unit": UNIT, "cores": threads, "kind": "port",
            "prompts": kind, "seconds": spent, "rounds": rounds, "ms_per_round": 1e3 * spent / max(rounds, 1),
            "sample": f"oracle/lmsd.py fp32 (reference SD control flow over the builder's fp32 Llama oracle; "
                      f"the reference has no transformer), first {nreq} requests of the same backlog run to "
                      f"completion one at a time (per-request engine API): {prefill_tok} prompt tokens "
                      f"prefilled, {rounds} rounds, {tok} tokens committed in {spent:.1f} s, k={args.k}"}


def llama_reference(args, rank, world):
    if rank != 0:
        return
    desc = llama_desc(args.workload)
    cb = llama_cpu_sample(desc, args, budget_s=args.cpu_budget)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_round"],
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic prompts (synth_prompt), random-init weights",
            "config": llama_config(args, world, args.batch),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ toy workload (config 2)
def toy_ours(args, rank, world, local_rank):
    import torch

    from paper_2604_20503_b200 import engine
    torch.cuda.set_device(local_rank)
    B = args.batch
    n_req = B * (args.steps + args.warmup) // 3 + 2 * B
    base = rank * n_req
    prompts, outl = prompts_for(base, n_req, 64, (4, 12), (16, 48))
    eng = engine.ServingEngine(abi.ToyParams.default(), max_batch=B, max_seq_len=128,
                               mode=abi.MODE_VSD_AD_EE, device=local_rank)
    for i, (p, m) in enumerate(zip(prompts, outl)):
        eng.submit(base + i, p, m)
    pol = abi.ExitPolicy.default()

    def run(n):
        # the serving loop in one native call (faser_serve_rounds): per round the seeded dynamic
        # k_i (sched_k), the Eq.5-10 gate plan, one step; no Python between rounds
        tok, _ = eng.serve_rounds(n, 7, base, pol, 0.7, 0.5, 32)
        return tok

    run(args.warmup)
    stream = torch.cuda.ExternalStream(eng.stream_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    t0 = time.perf_counter()
    tokens = run(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_ms = ev0.elapsed_time(ev1)
    eng.close()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": tokens / (dev_ms / 1e3), "unit": UNIT,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64/u64",
                          "data": "synthetic",
                          "config": {"workload": "config 2: toy pair, B=32, dynamic k, early exit",
                                     "global_batch": B * world},
                          "e2e": {"value": tokens / wall, "unit": UNIT}}), flush=True)


def toy_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import pyoracle as po
    if not os.path.exists(po.REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    R = po.ref()
    threads = max(1, min(os.cpu_count() or 1, args.batch))
    n = 40 * args.batch
    inl, outl = lens(1, n, (4, 12), (16, 48))
    prompts = [R.synth_prompt(1, i, inl[i], 64) for i in range(n)]
    cfg = abi.EpisodeCfg(model=abi.ToyParams.default(), max_batch=args.batch, early_exit=1, k_mode=1,
                         fixed_k=4, exempt_rule=1, threads=threads, k_seed=7,
                         max_rounds=args.steps + args.warmup, policy=abi.ExitPolicy.default(),
                         gate=abi.GatePlan(8, 32, 1.0))
    _, _, st = R.run_episode(cfg, prompts, outl)
    v = st.committed / st.wall_s
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0,
                      "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64/u64", "data": "synthetic",
                      "config": {"workload": "config 2: toy pair (reference engine)", "global_batch": args.batch},
                      "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                       "sample": f"{st.rounds} rounds"},
                      "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg4", "cfg5", "tiny", "tp_tiny", "toy"])
    ap.add_argument("--tp", action="store_true", help="tensor-parallel verification over the launched ranks")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--mode", default="vsd", choices=["vsd", "ad", "ee", "ov", "full", "vsd_ee"])
    ap.add_argument("--temperature", type=float, default=0.0,
                    help="> 0: sampling acceptance (coupled Gumbel-max, faser_set_sampling); 0: greedy")
    ap.add_argument("--chunk", type=int, default=0, help="overlap chunk (0: plan_overlap decides)")
    ap.add_argument("--gate-layer", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the embedded batch sweep")
    ap.add_argument("--recovery", action="store_true",
                    help="EE modes: recovery on prune (exempt_rule 2, beyond the reference's semantics)")
    ap.add_argument("--no-prefill-lane", action="store_true",
                    help="prefill admissions in the step itself instead of on the side lane")
    ap.add_argument("--trace", type=float, default=0.0,
                    help="replay a bursty arrival trace of this many seconds instead of a fixed backlog")
    ap.add_argument("--trace-rate", type=float, default=26.0, help="mean arrival rate (req/s) of --trace")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("FASER_BENCH_SHARE_GPU") == "1":
        # functional check of the N > 1 launcher path on a one-GPU box: every rank's replica on
        # cuda:0, metric reduction over gloo (NCCL refuses two ranks on one GPU). Not a
        # performance number: the replicas share one GPU.
        local_rank = 0
    if args.workload == "toy":
        (toy_reference if args.impl == "reference" else lambda a, r, w: toy_ours(a, r, w, local_rank))(args, rank, world)
    elif args.impl == "reference":
        llama_reference(args, rank, world)
    elif args.trace > 0:
        llama_trace(args, rank, world, local_rank)
    elif args.tp or args.workload == "cfg5":
        llama_tp(args, rank, world, local_rank)
    else:
        llama_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

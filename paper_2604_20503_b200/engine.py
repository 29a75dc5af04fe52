"""Python mirror of the C ABI (include/faser/engine.h) over ``libfaser_b200.so``.

Names follow the reference's C++ API so tests read like the reference's own:
  * ``LayeredToyLM``      — toylm.hpp:40-87 (final_and_noise, target_logits, target_next,
                            draft_next), batched over a ragged set of prefixes;
  * ``SpeculativeEngine`` — sdcore.hpp:81-116 (draft_tokens, full_verify,
                            verify_with_early_exit), batched over requests;
  * ``ServingEngine``     — the stateful submit/step engine that replaces the serving loop.
Every call runs the CUDA kernels; if the library (or a GPU) is missing the call raises —
there is no CPU fallback anywhere in this package.
"""
import ctypes as C
import os

import numpy as np

from . import abi

_LIB = None
# FASER_LIB: an alternative build of the same library (compile-time A/B variants, tools/build_variant.py)
LIB_PATH = os.environ.get("FASER_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfaser_b200.so")


class FaserError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{abi.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load the product library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.faser_last_error.restype = C.c_char_p
        L.faser_last_error.argtypes = [C.c_void_p]
        L.faser_kernel_launches.restype = C.c_int64
        L.faser_kernel_launches.argtypes = [C.c_void_p]
        L.faser_pending_work.restype = C.c_int32
        L.faser_pending_work.argtypes = [C.c_void_p]
        L.faser_engine_stream.restype = C.c_void_p
        L.faser_engine_stream.argtypes = [C.c_void_p]
        L.faser_engine_destroy.argtypes = [C.c_void_p]
        L.faser_engine_destroy.restype = None
        L.faser_drafter_destroy.argtypes = [C.c_void_p]
        L.faser_drafter_destroy.restype = None
        L.faser_drafter_beta.restype = C.c_double
        _LIB = L
    return _LIB


def _check(rc, engine=None):
    if rc != 0:
        msg = lib().faser_last_error(engine)
        raise FaserError(rc, msg.decode() if msg else "")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _ragged(rows):
    off = np.zeros(len(rows) + 1, np.int64)
    for i, r in enumerate(rows):
        off[i + 1] = off[i] + len(r)
    flat = np.zeros(max(int(off[-1]), 1), np.int32)
    for i, r in enumerate(rows):
        flat[off[i]:off[i + 1]] = r
    return flat, off


class LayeredToyLM:
    """GPU LayeredToyLM (toylm.hpp:40-87); every method takes a list of prefixes."""

    def __init__(self, params=None):
        self.params = params if params is not None else abi.ToyParams.default()

    @property
    def vocab_size(self):
        return self.params.vocab

    @property
    def eos_token(self):
        return self.params.vocab - 1

    def final_and_noise(self, prefixes):
        tok, off = _ragged(prefixes)
        V = self.params.vocab
        zf = np.zeros((len(prefixes), V), np.float64)
        zn = np.zeros_like(zf)
        _check(lib().faser_toy_final_and_noise(C.byref(self.params), len(prefixes), _ptr(tok),
                                               _ptr(off), _ptr(zf), _ptr(zn)))
        return zf, zn

    def target_logits(self, prefixes, layers):
        tok, off = _ragged(prefixes)
        lay = np.ascontiguousarray(np.broadcast_to(layers, (len(prefixes),)), np.int32)
        z = np.zeros((len(prefixes), self.params.vocab), np.float64)
        _check(lib().faser_toy_target_logits(C.byref(self.params), len(prefixes), _ptr(tok),
                                              _ptr(off), _ptr(lay), _ptr(z)))
        return z

    def _next(self, fn, prefixes):
        tok, off = _ragged(prefixes)
        out = np.zeros(len(prefixes), np.int32)
        _check(fn(C.byref(self.params), len(prefixes), _ptr(tok), _ptr(off), _ptr(out)))
        return out

    def target_next(self, prefixes):
        return self._next(lib().faser_toy_target_next, prefixes)

    def draft_next(self, prefixes):
        return self._next(lib().faser_toy_draft_next, prefixes)


class SpeculativeEngine:
    """GPU SpeculativeEngine (sdcore.hpp:81-116), batched: request i is described by its
    context (prompt ++ committed), |committed| and exempt_position."""

    def __init__(self, model):
        self.model = model

    def draft_tokens(self, contexts, s, remaining):
        tok, off = _ragged(contexts)
        n = len(contexts)
        s = np.ascontiguousarray(np.broadcast_to(s, (n,)), np.int32)
        rem = np.ascontiguousarray(np.broadcast_to(remaining, (n,)), np.int32)
        out = np.zeros((n, abi.MAX_SPEC), np.int32)
        ol = np.zeros(n, np.int32)
        _check(lib().faser_toy_draft_tokens(C.byref(self.model.params), n, _ptr(tok), _ptr(off),
                                            _ptr(s), _ptr(rem), _ptr(out), _ptr(ol)))
        return [out[i, :ol[i]].tolist() for i in range(n)]

    def _verify(self, contexts, drafted, committed_len, exempt, policy, gate):
        tok, off = _ragged(contexts)
        n = len(contexts)
        cl = np.ascontiguousarray(np.broadcast_to(committed_len, (n,)), np.int32)
        ex = np.ascontiguousarray(np.broadcast_to(exempt, (n,)), np.int32)
        d = np.zeros((n, abi.MAX_SPEC), np.int32)
        dl = np.zeros(n, np.int32)
        for i, r in enumerate(drafted):
            d[i, :len(r)] = r
            dl[i] = len(r)
        out = (abi.VerifyOutcome * max(n, 1))()
        pol = policy or abi.ExitPolicy.default()
        _check(lib().faser_toy_verify(C.byref(self.model.params), n, _ptr(tok), _ptr(off), _ptr(cl),
                                      _ptr(ex), _ptr(d), _ptr(dl), C.byref(pol),
                                      C.byref(gate) if gate is not None else None, out))
        return list(out[:n])

    def full_verify(self, contexts, drafted):
        return self._verify(contexts, drafted, 0, -1, None, None)

    def verify_with_early_exit(self, contexts, drafted, policy, gate, committed_len, exempt=-1):
        return self._verify(contexts, drafted, committed_len, exempt, policy, gate)


def synth_prompt(seed, index, length, vocab):
    """synth_prompt (workload.cpp:116-122): seeded prompt tokens in [0, vocab-2] (never EOS)."""
    buf = np.zeros(max(int(length), 1), np.int32)
    _check(lib().faser_synth_prompt(C.c_uint64(seed), int(index), int(length), int(vocab), _ptr(buf)))
    return buf.tolist()


class TpGroup:
    """Tensor-parallel group handle (faser_tp_group): ``TpGroup.local(n)`` = n in-process ranks on
    one device (each rank's engine stepped from its own thread), ``TpGroup.nccl(uid, n, rank,
    device)`` = one process per GPU over NCCL (uid from ``TpGroup.nccl_unique_id()`` on rank 0)."""

    def __init__(self, h, size):
        self.h, self.size = h, size

    @classmethod
    def local(cls, size):
        h = C.c_void_p()
        _check(lib().faser_tp_local_group_create(int(size), C.byref(h)))
        return cls(h, size)

    @staticmethod
    def nccl_unique_id():
        buf = (C.c_uint8 * 128)()
        _check(lib().faser_tp_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, uid, size, rank, device):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().faser_tp_nccl_group_create(buf, int(size), int(rank), int(device), C.byref(h)))
        return cls(h, size)

    def close(self):
        if self.h:
            lib().faser_tp_group_destroy(self.h)
            self.h = None


def default_engine_cfg(**kw):
    cfg = abi.EngineCfg(device=0, max_batch=256, max_seq_len=4096, mode=abi.MODE_VSD,
                        default_spec_length=4, exempt_rule=1,
                        exit_policy=abi.ExitPolicy.default(), max_pending=1 << 20,
                        pending_tokens=1 << 24)
    for k, v in kw.items():
        if k == "tp_group" and isinstance(v, TpGroup):
            v = v.h
        setattr(cfg, k, v)
    return cfg


def k_table(policy, num_layers):
    t = (C.c_int32 * (abi.MAX_LAYERS + 1))()
    _check(lib().faser_k_table(C.byref(policy), num_layers, t))
    return t


def make_gate_plan(policy, entries, b, r, num_layers, models=None):
    arr = (abi.GateEntry * max(len(entries), 1))()
    for i, (s, a) in enumerate(entries):
        arr[i].spec_length = s
        arr[i].accept_estimate = a
    g = abi.GatePlan()
    _check(lib().faser_make_gate_plan(C.byref(policy), arr, len(entries), C.c_double(b),
                                      C.c_double(r), C.byref(models) if models else None,
                                      num_layers, C.byref(g)))
    return g


def plan_overlap(s, b, r_grid=(0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9), models=None):
    """plan_overlap (overlap.cpp:23-42): chunk / SM share that beats the serial estimate, if any."""
    rg = np.ascontiguousarray(r_grid, np.float64)
    out = abi.OverlapPlan()
    _check(lib().faser_plan_overlap(int(s), int(b), C.byref(models) if models else None, _ptr(rg), len(rg),
                                    C.byref(out)))
    return out


def num_sms(device=0):
    """SM count of `device` (the lanes partition it in multiples of 8)."""
    import torch
    return torch.cuda.get_device_properties(device).multi_processor_count


class ServingEngine:
    """Stateful GPU engine: submit() requests, step() one draft->verify->commit round."""

    def __init__(self, model_params=None, cfg=None, desc=None, **cfg_kw):
        """Toy engine from ``model_params`` (LayeredToyLM::Params), or a Llama-style engine
        from ``desc`` (abi.ModelDesc with kind MODEL_LLAMA, see llama.py presets)."""
        self.h = None
        self.params = model_params if model_params is not None else abi.ToyParams.default()
        self.cfg = cfg if cfg is not None else default_engine_cfg(**cfg_kw)
        if desc is None:
            desc = abi.ModelDesc(kind=abi.MODEL_TOY, toy=self.params)
        self.desc = desc
        h = C.c_void_p()
        _check(lib().faser_engine_create(C.byref(desc), C.byref(self.cfg), C.byref(h)))
        self.h = h
        self._res = (abi.RoundResult * self.cfg.max_batch)()
        self.plan = abi.StepPlan()
        self.plan.gate = abi.GatePlan(self.cfg.exit_policy.l_init, self.cfg.exit_policy.l_init, 1.0)

    def close(self):
        if self.h:
            lib().faser_engine_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def submit(self, req_id, prompt, max_out):
        p = np.ascontiguousarray(prompt, np.int32)
        _check(lib().faser_submit(self.h, C.c_int64(req_id), _ptr(p), len(p), max_out), self.h)

    def set_spec_lengths(self, ids, ks):
        ids = np.ascontiguousarray(ids, np.int64)
        ks = np.ascontiguousarray(ks, np.int32)
        _check(lib().faser_set_spec_lengths(self.h, _ptr(ids), _ptr(ks), len(ids)), self.h)

    def live_requests(self):
        buf = np.zeros(self.cfg.max_batch, np.int64)
        n = C.c_int32()
        _check(lib().faser_live_requests(self.h, _ptr(buf), len(buf), C.byref(n)), self.h)
        return buf[:n.value].tolist()

    def set_gate(self, gate):
        self.plan.gate = gate

    def set_overlap(self, enabled, chunk=2, r=0.5):
        """OverlapPlan (overlap.hpp:11-17): in MODE_FULL, frontier chunk q of the drafted tokens
        is verified on a second lane while chunk q+1 is drafted."""
        self.plan.overlap = abi.OverlapPlan(1 if enabled else 0, chunk, r, 0.0, 0.0)
        self.overlap_state = (bool(enabled), chunk, r)

    def set_lane_mode(self, mode):
        """abi.LANES_OVERLAP (default) or abi.LANES_ISOLATED: the same partitions and chunks with the
        lanes serialised (draft chunk q+1 after verify chunk q), the interference baseline."""
        self.plan.lane_mode = int(mode)

    def last_timeline(self, cap=4 * (abi.MAX_SPEC + 2)):
        """Measured PipelineTimeline of the last overlapped step: (TimelineInfo, [TimelineEvent])."""
        evs = (abi.TimelineEvent * cap)()
        info = abi.TimelineInfo()
        _check(lib().faser_last_timeline(self.h, evs, cap, C.byref(info)), self.h)
        return info, [evs[i] for i in range(min(cap, info.n_events))]

    def step(self):
        n = C.c_int32()
        _check(lib().faser_step(self.h, C.byref(self.plan), self._res, self.cfg.max_batch,
                                C.byref(n)), self.h)
        return self._res[:n.value]

    def committed(self, req_id, cap=1 << 16):
        buf = np.zeros(cap, np.int32)
        n = C.c_int32()
        _check(lib().faser_get_committed(self.h, C.c_int64(req_id), _ptr(buf), cap, C.byref(n)),
               self.h)
        return buf[:n.value].tolist()

    def pending_work(self):
        return lib().faser_pending_work(self.h)

    def last_step_timing(self):
        a, b, c = C.c_float(), C.c_float(), C.c_float()
        _check(lib().faser_last_step_timing(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def serve_rounds(self, n_rounds, seed, id_base=0, policy=None, accept_est=0.7, r=0.5, num_layers=32):
        """The sim loop in one native call (faser_serve_rounds): per round k_i = sched_k(seed,
        req_id - id_base, rounds served), set_spec_lengths, make_gate_plan when `policy` is
        given, step. Returns (committed tokens, rounds executed)."""
        tok, rnd = C.c_int64(), C.c_int32()
        _check(lib().faser_serve_rounds(self.h, int(n_rounds), C.c_uint64(seed), C.c_int64(id_base),
                                        C.byref(policy) if policy is not None else None, C.c_double(accept_est),
                                        C.c_double(r), int(num_layers), C.byref(tok), C.byref(rnd)), self.h)
        return tok.value, rnd.value

    def set_sampling(self, temperature, seed=0):
        """Coupled Gumbel-max sampling at `temperature` (0 = greedy); faser_set_sampling."""
        _check(lib().faser_set_sampling(self.h, C.c_double(temperature), C.c_uint64(seed)), self.h)

    def debug_set_skip_mask(self, mask):
        """Timing experiments only: kernel classes the following steps skip (results invalid)."""
        _check(lib().faser_debug_set_skip_mask(self.h, int(mask)), self.h)

    def set_prefill_lane(self, on):
        _check(lib().faser_set_prefill_lane(self.h, 1 if on else 0), self.h)

    def join_lanes(self):
        """Engine stream waits for the admission-prefill lane (before a closing timing event)."""
        _check(lib().faser_engine_join_lanes(self.h), self.h)

    def last_step_prefill_ms(self):
        """Admission + prefill part of the last step's draft-lane time (ms)."""
        a = C.c_float()
        _check(lib().faser_last_step_prefill(self.h, C.byref(a)))
        return a.value

    def last_step_bytes(self):
        a, b = C.c_int64(), C.c_int64()
        _check(lib().faser_last_step_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stream_ptr(self):
        return lib().faser_engine_stream(self.h)

    def kernel_launches(self):
        return lib().faser_kernel_launches(self.h)

    # ---- per-kernel-class device timing (CUDA events around launches)
    KERNEL_CLASSES = ("verify_gemm", "verify_attention", "draft_gemm", "draft_attention", "verify_lm_head")

    def set_kernel_timing(self, enabled):
        _check(lib().faser_set_kernel_timing(self.h, 1 if enabled else 0), self.h)

    def kernel_stats(self):
        out = {}
        for i, name in enumerate(self.KERNEL_CLASSES):
            ms, n, b = C.c_double(), C.c_int64(), C.c_double()
            _check(lib().faser_kernel_stats(self.h, i, C.byref(ms), C.byref(n), C.byref(b)), self.h)
            f = C.c_double()
            _check(lib().faser_kernel_flops(self.h, i, C.byref(f)), self.h)
            out[name] = {"ms": ms.value, "launches": n.value, "bytes": b.value, "flops": f.value}
        return out

    # ---- Llama validation hooks (cfg.debug_capture = 1)
    def debug_verify_logits(self, stage=0):
        """(logits [rows][V] float32, ids [rows][2] = (req_id, j)) of the last step's verify
        forward: stage 0 = final, stage l = gated layer l."""
        V = self.desc.target.vocab
        rows = C.c_int32()
        _check(lib().faser_debug_verify_logits(self.h, stage, None, None, 0, C.byref(rows)), self.h)
        n = rows.value
        z = np.zeros((max(n, 1), V), np.float32)
        ids = np.zeros((max(n, 1), 2), np.int64)
        _check(lib().faser_debug_verify_logits(self.h, stage, _ptr(z), _ptr(ids), n, C.byref(rows)),
               self.h)
        return z[:n], ids[:n]

    def debug_drafted(self):
        n = C.c_int32()
        buf = np.zeros((self.cfg.max_batch, abi.MAX_SPEC), np.int32)
        _check(lib().faser_debug_drafted(self.h, _ptr(buf), self.cfg.max_batch, C.byref(n)), self.h)
        return buf[:n.value]

    def debug_weights(self, model, which, layer, offset, n):
        out = np.zeros(max(n, 1), np.uint16)
        _check(lib().faser_debug_weights(self.h, model, which, layer, C.c_int64(offset), n, _ptr(out)),
               self.h)
        return out[:n]

    def debug_kv_pages(self, req_id):
        buf = np.zeros(4096, np.int32)
        n = C.c_int32()
        _check(lib().faser_debug_kv_pages(self.h, C.c_int64(req_id), _ptr(buf), len(buf), C.byref(n)),
               self.h)
        return buf[:n.value].tolist()

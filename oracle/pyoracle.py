"""oracle/pyoracle.py — TEST INFRASTRUCTURE ONLY.

ctypes loaders for the two CPU oracles:
  * ``ref()``      -> oracle/_ref/libspecsim_ref.so  (the reference's own TUs, symbols specref_*)
  * ``restated()`` -> oracle/_build/liboracle.so     (plain-C restatement, symbols oracle_*)
Both expose the same call shapes; ``Oracle`` wraps either with numpy-friendly methods.
Only tests/, __graft_entry__.smoke() and bench.py's baseline legs import this module.
"""
import ctypes as C
import os

import numpy as np

from paper_2604_20503_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libspecsim_ref.so")
RESTATED_SO = os.path.join(HERE, "_build", "liboracle.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def ragged(rows):
    """List of token lists -> (flat int32 tokens, int64 offsets[n+1])."""
    off = np.zeros(len(rows) + 1, np.int64)
    for i, r in enumerate(rows):
        off[i + 1] = off[i] + len(r)
    flat = np.zeros(max(int(off[-1]), 1), np.int32)
    for i, r in enumerate(rows):
        flat[off[i]:off[i + 1]] = r
    return flat, off


class Oracle:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (build())")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.kind = "reference" if prefix == "specref_" else "port"

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # ---------------------------------------------------------------- row ops
    def final_and_noise(self, p, rows):
        tok, off = ragged(rows)
        zf = np.zeros((len(rows), p.vocab), np.float64)
        zn = np.zeros_like(zf)
        rc = self.fn("final_and_noise")(C.byref(p), len(rows), tok.ctypes.data_as(C.c_void_p),
                                        off.ctypes.data_as(C.c_void_p),
                                        zf.ctypes.data_as(C.c_void_p), zn.ctypes.data_as(C.c_void_p))
        assert rc == 0, rc
        return zf, zn

    def target_logits(self, p, rows, layers):
        tok, off = ragged(rows)
        lay = np.ascontiguousarray(layers, np.int32)
        z = np.zeros((len(rows), p.vocab), np.float64)
        rc = self.fn("target_logits")(C.byref(p), len(rows), tok.ctypes.data_as(C.c_void_p),
                                      off.ctypes.data_as(C.c_void_p), lay.ctypes.data_as(C.c_void_p),
                                      z.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError(abi.STATUS_NAMES[rc])
        return z

    def _next(self, name, p, rows):
        tok, off = ragged(rows)
        out = np.zeros(len(rows), np.int32)
        rc = self.fn(name)(C.byref(p), len(rows), tok.ctypes.data_as(C.c_void_p),
                           off.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        assert rc == 0, rc
        return out

    def target_next(self, p, rows):
        return self._next("target_next", p, rows)

    def draft_next(self, p, rows):
        return self._next("draft_next", p, rows)

    def autoregressive_decode(self, p, prompt, max_out):
        pr = np.ascontiguousarray(prompt, np.int32)
        out = np.zeros(max(max_out, 1), np.int32)
        n = C.c_int32()
        rc = self.fn("autoregressive_decode")(C.byref(p), pr.ctypes.data_as(C.c_void_p), len(pr),
                                              max_out, out.ctypes.data_as(C.c_void_p), C.byref(n))
        assert rc == 0, rc
        return out[:n.value].tolist()

    def draft_tokens(self, p, rows, s, remaining):
        tok, off = ragged(rows)
        s = np.ascontiguousarray(s, np.int32)
        rem = np.ascontiguousarray(remaining, np.int32)
        out = np.zeros((len(rows), abi.MAX_SPEC), np.int32)
        ol = np.zeros(len(rows), np.int32)
        rc = self.fn("draft_tokens")(C.byref(p), len(rows), tok.ctypes.data_as(C.c_void_p),
                                     off.ctypes.data_as(C.c_void_p), s.ctypes.data_as(C.c_void_p),
                                     rem.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p),
                                     ol.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError(abi.STATUS_NAMES[rc])
        return [out[i, :ol[i]].tolist() for i in range(len(rows))]

    def verify(self, p, rows, committed_len, exempt, drafted, policy=None, gate=None, k_table=None):
        tok, off = ragged(rows)
        n = len(rows)
        cl = np.ascontiguousarray(committed_len, np.int32)
        ex = np.ascontiguousarray(exempt, np.int32)
        d = np.zeros((n, abi.MAX_SPEC), np.int32)
        dl = np.zeros(n, np.int32)
        for i, r in enumerate(drafted):
            d[i, :len(r)] = r
            dl[i] = len(r)
        out = (abi.VerifyOutcome * n)()
        pol = policy or abi.ExitPolicy.default()
        args = [C.byref(p), n, tok.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p),
                cl.ctypes.data_as(C.c_void_p), ex.ctypes.data_as(C.c_void_p),
                d.ctypes.data_as(C.c_void_p), dl.ctypes.data_as(C.c_void_p), C.byref(pol),
                C.byref(gate) if gate is not None else None]
        if self.prefix == "oracle_":
            kt = None if k_table is None else np.ascontiguousarray(k_table, np.int32)
            args.append(kt.ctypes.data_as(C.c_void_p) if kt is not None else None)
        else:
            assert k_table is None, "reference verify uses ExitPolicy::k_at"
        rc = self.fn("verify")(*args, out)
        assert rc == 0, rc
        return list(out)

    def k_at(self, policy, layer, num_layers):
        if self.prefix == "oracle_":
            self.lib.oracle_k_at.restype = C.c_int
            return self.lib.oracle_k_at(C.byref(policy), layer, num_layers)
        out = C.c_int32()
        assert self.lib.specref_k_at(C.byref(policy), layer, num_layers, C.byref(out)) == 0
        return out.value

    def token_exit_test(self, z, d, k):
        z = np.ascontiguousarray(z, np.float64)
        if self.prefix == "oracle_":
            return bool(self.lib.oracle_token_exit_test(z.ctypes.data_as(C.c_void_p), len(z), d, k))
        out = C.c_int32()
        assert self.lib.specref_token_exit_test(z.ctypes.data_as(C.c_void_p), len(z), d, k,
                                                C.byref(out)) == 0
        return bool(out.value)

    def synth_prompt(self, seed, index, length, vocab):
        out = np.zeros(max(length, 1), np.int32)
        rc = self.fn("synth_prompt")(C.c_uint64(seed), index, length, vocab,
                                     out.ctypes.data_as(C.c_void_p))
        assert rc == 0
        return out.tolist()

    def run_episode(self, cfg, prompts, max_out, log_cap=0):
        """Serving loop over a backlog. Returns (outputs, round_log, stats)."""
        tok, off = ragged(prompts)
        mo = np.ascontiguousarray(max_out, np.int32)
        n = len(prompts)
        cap = int(mo.max()) if n else 1
        out = np.zeros((n, max(cap, 1)), np.int32)
        ol = np.zeros(n, np.int32)
        log = (abi.RoundResult * max(log_cap, 1))()
        n_log = C.c_int64()
        st = abi.EpisodeStats()
        cfg.n_requests = n
        rc = self.fn("run_episode")(C.byref(cfg), tok.ctypes.data_as(C.c_void_p),
                                    off.ctypes.data_as(C.c_void_p), mo.ctypes.data_as(C.c_void_p),
                                    out.ctypes.data_as(C.c_void_p), max(cap, 1),
                                    ol.ctypes.data_as(C.c_void_p), log if log_cap else None,
                                    log_cap, C.byref(n_log), C.byref(st))
        if rc:
            raise ValueError(abi.STATUS_NAMES[rc])
        outs = [out[i, :ol[i]].tolist() for i in range(n)]
        return outs, list(log[:min(n_log.value, log_cap)]) if log_cap else [], st


_cache = {}


def ref():
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_SO, "specref_")
    return _cache["ref"]


def restated():
    if "port" not in _cache:
        _cache["port"] = Oracle(RESTATED_SO, "oracle_")
    return _cache["port"]


def backlog_lengths(seed, n, in_range=(4, 12), out_range=(16, 48)):
    """lens substream of synth_workload (workload.cpp:77,89-90) for n backlog records."""
    lib = restated().lib
    a = np.zeros(n, np.int32)
    b = np.zeros(n, np.int32)
    lib.oracle_backlog_lengths(C.c_uint64(seed), n, in_range[0], in_range[1], out_range[0],
                               out_range[1], a.ctypes.data_as(C.c_void_p),
                               b.ctypes.data_as(C.c_void_p))
    return a.tolist(), b.tolist()

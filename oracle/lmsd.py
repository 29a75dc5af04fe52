"""TEST INFRASTRUCTURE ONLY — the reference's speculative-decoding semantics over the fp32
oracle models (oracle/llama_oracle.c), for configs 3-5.

Follows the reference's control flow exactly, with the transformer pair in place of
LayeredToyLM:
  draft_tokens   sdcore.cpp:45-59   (budget min(s, max_out - |committed|), EOS stop)
  full_verify    sdcore.cpp:61-81   (longest matching prefix; recovery = target argmax at the
                                     first mismatch; no bonus token on full acceptance)
  commit         sdcore.cpp:182-197 (accepted then recovery; done at EOS or max_out)
argmax ties -> lowest id (argmax_lowest, toylm.cpp:9-16; numpy argmax returns the first max).
Used as the CPU baseline of bench.py (`cpu_baseline.kind = "port"`, the reference has no
transformer path) and by the parity tests.
"""
import numpy as np

from . import lmoracle


class Request:
    def __init__(self, rid, prompt, max_out):
        self.id = rid
        self.prompt = list(prompt)
        self.committed = []
        self.max_out = max_out
        self.done = max_out == 0

    @property
    def ctx(self):
        return self.prompt + self.committed


class OracleSD:
    """Greedy SD over (draft, target) oracle models with incremental KV caches per request."""

    def __init__(self, desc, threads=None):
        self.desc = desc
        self.V = desc.target.vocab
        self.eos = self.V - 1
        self.draft = lmoracle.Model(desc.draft, desc.bigram_a, desc.bigram_b, threads)
        self.target = lmoracle.Model(desc.target, desc.bigram_a, desc.bigram_b, threads)
        self.reqs = {}
        self.caches = {}

    def submit(self, rid, prompt, max_out, cap=4096):
        L = lmoracle.lib()
        r = Request(rid, prompt, max_out)
        self.reqs[rid] = r
        cd = L.lmo_cache_create(self.draft.h, cap)
        ct = L.lmo_cache_create(self.target.h, cap)
        self.caches[rid] = (cd, ct)
        if len(prompt) > 1:  # caches hold positions [0, len-1): the last token is pending
            tok = np.ascontiguousarray(prompt[:-1], np.int32)
            assert L.lmo_forward(self.draft.h, cd, lmoracle._p(tok), len(tok), None, 0, None) == 0
            assert L.lmo_forward(self.target.h, ct, lmoracle._p(tok), len(tok), None, 0, None) == 0
        return r

    def _step(self, model, cache, tokens, layers=None):
        L = lmoracle.lib()
        tok = np.ascontiguousarray(tokens, np.int32)
        lay = np.asarray(layers or [model.shape.layers], np.int32)
        out = np.zeros((len(lay), len(tok), self.V), np.float32)
        assert L.lmo_forward(model.h, cache, lmoracle._p(tok), len(tok), lmoracle._p(lay), len(lay),
                             lmoracle._p(out)) == 0
        return out

    def draft_tokens(self, rid, s):
        """sdcore.cpp:45-59."""
        r = self.reqs[rid]
        assert not r.done and s >= 1
        cd, _ = self.caches[rid]
        budget = min(s, r.max_out - len(r.committed))
        out = []
        cur = r.ctx[-1]
        for _ in range(budget):
            z = self._step(self.draft, cd, [cur])[0, 0]
            cur = int(np.argmax(z))
            out.append(cur)
            if cur == self.eos:
                break
        return out

    def verify_logits(self, rid, drafted):
        """Target logits of the verify rows [ctx[-1], d0 .. d_{k-2}] (row j predicts d_j)."""
        _, ct = self.caches[rid]
        r = self.reqs[rid]
        return self._step(self.target, ct, [r.ctx[-1]] + list(drafted[:-1]))[0]

    def full_verify(self, rid, drafted, logits=None):
        """sdcore.cpp:61-81 -> (accepted, recovery or None)."""
        z = self.verify_logits(rid, drafted) if logits is None else logits
        acc = 0
        for j, d in enumerate(drafted):
            t = int(np.argmax(z[j]))
            if d == t:
                acc += 1
            else:
                return acc, t
        return acc, None

    def commit(self, rid, drafted, acc, rec):
        """sdcore.cpp:182-197, then roll both caches back to positions [0, len-1)."""
        L = lmoracle.lib()
        r = self.reqs[rid]
        c = 0
        for d in drafted[:acc]:
            if r.done:
                break
            r.committed.append(d)
            c += 1
            if d == self.eos or len(r.committed) == r.max_out:
                r.done = True
        if rec is not None and not r.done:
            r.committed.append(rec)
            c += 1
            if rec == self.eos or len(r.committed) == r.max_out:
                r.done = True
        keep = len(r.ctx) - 1
        for cache in self.caches[rid]:
            assert L.lmo_cache_truncate(cache, min(keep, L.lmo_cache_len(cache))) == 0
        return c

    def round(self, rid, s):
        d = self.draft_tokens(rid, s)
        acc, rec = self.full_verify(rid, d)
        return d, acc, rec, self.commit(rid, d, acc, rec)

    def release(self, rid):
        """Frees a finished request's KV caches."""
        L = lmoracle.lib()
        for c in self.caches.pop(rid, ()):
            L.lmo_cache_destroy(c)

    def close(self):
        L = lmoracle.lib()
        for cd, ct in self.caches.values():
            L.lmo_cache_destroy(cd)
            L.lmo_cache_destroy(ct)
        self.caches = {}
        self.draft.close()
        self.target.close()

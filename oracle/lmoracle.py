"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/llama_oracle.c (fp32 CPU forward of the
Llama-style random-init models; builder-written oracle, the reference has no transformer).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this."""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libllama_oracle.so")
_L = None


def lib():
    global _L
    if _L is None:
        L = C.CDLL(SO)
        L.lmo_create.restype = C.c_void_p
        L.lmo_create.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
        L.lmo_destroy.argtypes = [C.c_void_p]
        L.lmo_cache_create.restype = C.c_void_p
        L.lmo_cache_create.argtypes = [C.c_void_p, C.c_int]
        L.lmo_cache_destroy.argtypes = [C.c_void_p]
        L.lmo_cache_truncate.argtypes = [C.c_void_p, C.c_int]
        L.lmo_cache_len.argtypes = [C.c_void_p]
        L.lmo_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                  C.c_void_p]
        L.lmo_greedy.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                 C.c_void_p, C.c_void_p]
        L.lmo_weight.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_void_p]
        L.lmo_set_threads.argtypes = [C.c_int]
        L.lmo_weight_block.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_void_p]
        _L = L
    return _L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Model:
    """One fp32 oracle model built from an abi.LlamaShape and the bigram map (a, b)."""

    def __init__(self, shape, a, b, threads=None):
        lib().lmo_set_threads(threads or os.cpu_count() or 1)
        self.shape = shape
        self.h = lib().lmo_create(C.byref(shape), a, b)

    def close(self):
        if self.h:
            lib().lmo_destroy(self.h)
            self.h = None

    __del__ = close

    def weight(self, which, layer, idx):
        out = C.c_uint16()
        lib().lmo_weight(self.h, which, layer, idx, C.byref(out))
        return out.value

    def tensor(self, which, layer=0):
        """A whole bf16 tensor as uint16 [rows][cols] (which: 0 lm, 1 emb, 2 wqkv, 3 wo, 4 wgu
        (interleaved 64-row gate/up groups), 5 wd)."""
        s = self.shape
        d, F, V = s.d_model, s.ffn, s.vocab
        qkv = (s.n_heads + 2 * s.n_kv_heads) * s.head_dim
        qd = s.n_heads * s.head_dim
        rows, cols = {0: (V, d), 1: (V, d), 2: (qkv, d), 3: (d, qd), 4: (2 * F, d), 5: (d, F)}[which]
        out = np.zeros((rows, cols), np.uint16)
        assert lib().lmo_weight_block(self.h, which, layer, 0, rows * cols, _p(out)) == 0
        return out

    def logits(self, tokens, rows_from, layers=None):
        """Logits of positions rows_from..len(tokens)-1 after each layer count in `layers`
        (default: final). Returns [len(layers)][rows][V]."""
        s = self.shape
        layers = list(layers or [s.layers])
        tok = np.ascontiguousarray(tokens, np.int32)
        n = len(tok)
        cache = lib().lmo_cache_create(self.h, n + 1)
        lay = np.asarray(layers, np.int32)
        out = np.zeros((len(layers), n, s.vocab), np.float32)
        rc = lib().lmo_forward(self.h, cache, _p(tok), n, _p(lay), len(layers), _p(out))
        lib().lmo_cache_destroy(cache)
        assert rc == 0
        return out[:, rows_from:, :]

    def greedy(self, prompt, max_out, eos):
        p = np.ascontiguousarray(prompt, np.int32)
        out = np.zeros(max(max_out, 1), np.int32)
        n = C.c_int32()
        assert lib().lmo_greedy(self.h, _p(p), len(p), max_out, eos, _p(out), C.byref(n)) == 0
        return out[:n.value].tolist()

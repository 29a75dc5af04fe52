"""Host-side speculative-length controller (AdaptiveDrafter, drafter.hpp:98-129) over the C ABI.

The engine consumes k_i through faser_set_spec_lengths; this class produces them the way the
reference's serving loop does: assign_lengths before a step, observe_round after it.
"""
import ctypes as C

import numpy as np

from . import abi
from .engine import _check, _ptr, lib


class DrafterCfg(C.Structure):
    _fields_ = [("n_candidates", C.c_int32), ("candidates", C.c_int32 * 16),
                ("window_ctx", C.c_int32), ("window_request", C.c_int32), ("reserved0", C.c_int32),
                ("epsilon", C.c_double), ("kernel_len", C.c_double), ("kernel_var", C.c_double),
                ("noise_var", C.c_double), ("cold_start_accept", C.c_double)]

    @classmethod
    def default(cls):
        c = cls()
        lib().faser_drafter_default_cfg(C.byref(c))
        return c


class AdaptiveDrafter:
    def __init__(self, cfg=None, models=None):
        self.cfg = cfg if cfg is not None else DrafterCfg.default()
        h = C.c_void_p()
        _check(lib().faser_drafter_create(C.byref(self.cfg), C.byref(models) if models else None,
                                          C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().faser_drafter_destroy(self.h)
            self.h = None

    __del__ = close

    def set_models(self, models):
        """Installs refreshed stage-latency models (profiler.OnlineProfiler) for later rounds."""
        _check(lib().faser_drafter_set_models(self.h, C.byref(models)))

    def assign_lengths(self, req_ids, b, r):
        ids = np.ascontiguousarray(req_ids, np.int64)
        out = np.zeros(max(len(ids), 1), np.int32)
        _check(lib().faser_drafter_assign(self.h, _ptr(ids), len(ids), int(b), C.c_double(r), _ptr(out)))
        return out[:len(ids)].tolist()

    def observe_round(self, b, r, t_obs_ms, req_ids, spec, submitted, accepted):
        a = [np.ascontiguousarray(x, t) for x, t in ((req_ids, np.int64), (spec, np.int32),
                                                     (submitted, np.int32), (accepted, np.int32))]
        _check(lib().faser_drafter_observe(self.h, int(b), C.c_double(r), C.c_double(t_obs_ms),
                                           *[_ptr(x) for x in a], len(a[0])))

    def observe_results(self, results, b, r, t_obs_ms):
        """Feeds a faser_step result list (abi.RoundResult) back."""
        self.observe_round(b, r, t_obs_ms, [x.req_id for x in results], [x.spec_length for x in results],
                           [x.outcome.submitted for x in results],
                           [x.outcome.accepted_count for x in results])
        for x in results:
            if x.done:
                lib().faser_drafter_release(self.h, C.c_int64(x.req_id))

    def estimate(self, req_ids, ks, b, r):
        """AcceptanceBook::estimate per request at its assigned length (drafter.cpp:151-161)."""
        ids = np.ascontiguousarray(req_ids, np.int64)
        s = np.ascontiguousarray(ks, np.int32)
        out = np.zeros(max(len(ids), 1))
        _check(lib().faser_drafter_estimate(self.h, _ptr(ids), _ptr(s), len(ids), int(b), C.c_double(r), _ptr(out)))
        return out[:len(ids)].tolist()

    def request_window(self, req_id, qs):
        q = np.ascontiguousarray(qs, np.int32)
        out = np.zeros(len(q) + 1)
        _check(lib().faser_drafter_request_window(self.h, C.c_int64(req_id), _ptr(q), len(q), _ptr(out)))
        return out.tolist()

    def posterior(self, b, r):
        m = self.cfg.n_candidates
        mu = np.zeros(m)
        sd = np.zeros(m)
        n = C.c_int32()
        _check(lib().faser_drafter_posterior(self.h, int(b), C.c_double(r), _ptr(mu), _ptr(sd), C.byref(n)))
        return mu, sd, n.value

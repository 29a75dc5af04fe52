"""CPU tier: the reference's output wire formats (trace CSV, metrics JSON lines, summary CSV),
byte-for-byte against the reference's own writers and parser (oracle/_ref compiles
workload.cpp and metrics.cpp in place)."""
import ctypes as C
import os
import random

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2604_20503_b200 import metrics

needs_ref = pytest.mark.skipif(not os.path.exists(po.REF_SO), reason="oracle/_ref not built")


def _ref():
    return po.ref().lib


@needs_ref
def test_trace_csv_bytes_and_ingest_match_reference(tmp_path):
    rng = random.Random(5)
    recs = [(rng.uniform(0, 6e4), rng.randint(1, 2048), rng.randint(1, 512)) for _ in range(300)]
    recs += [(0.0, 0, 0), (1.0005, 7, 9), (123456.78951, 3, 4)]
    mine, theirs = tmp_path / "mine.csv", tmp_path / "ref.csv"
    metrics.write_trace(mine, recs)
    a = np.array([r[0] for r in recs])
    i = np.array([r[1] for r in recs], np.int32)
    o = np.array([r[2] for r in recs], np.int32)
    assert _ref().specref_write_trace(str(theirs).encode(), len(recs), a.ctypes.data_as(C.c_void_p),
                                      i.ctypes.data_as(C.c_void_p), o.ctypes.data_as(C.c_void_p)) == 0
    assert mine.read_bytes() == theirs.read_bytes()
    assert metrics.ingest_trace(theirs) == _ingest_ref(theirs)


def _ingest_ref(path):
    cap = 4096
    a, i, o, n = np.zeros(cap), np.zeros(cap, np.int32), np.zeros(cap, np.int32), C.c_int32()
    rc = _ref().specref_ingest_trace(str(path).encode(), cap, a.ctypes.data_as(C.c_void_p),
                                     i.ctypes.data_as(C.c_void_p), o.ctypes.data_as(C.c_void_p), C.byref(n))
    if rc != 0:
        return "error"
    return [(float(a[k]), int(i[k]), int(o[k])) for k in range(n.value)]


@needs_ref
@pytest.mark.parametrize("text", [
    "arrival_ms,input_len,output_len\n3.5,10,20\n1.25,4,8\n\n  \n2,1,1\n",   # header, blanks, unsorted
    "1,2,3\n0.5,2,3\n0.5,1,1\n",                                           # no header, stable ties
    " 1.0 , 2.9 , 3.99\n",                                                 # spaces, truncation to int
    "hdr\n1,2,3\nbad,row\n",                                                # malformed later row -> error
    "1,2,3,4\n5,6,7\n",                                                     # extra column on line 1 = header
    "1,2,3\n4,5,6 x\n",                                                     # trailing garbage -> error
    "1,-2,3\n",                                                             # negative -> header, empty
    "1e3,2,3\n",
])
def test_ingest_trace_edge_cases_match_reference(tmp_path, text):
    p = tmp_path / "t.csv"
    p.write_text(text)
    try:
        got = metrics.ingest_trace(p)
    except metrics.ParseError:
        got = "error"
    assert got == _ingest_ref(p)


def _random_summary(rng):
    s = metrics.MetricsSummary(mode=rng.choice(["VSD", "VSD_AD", "VSD_AD_EE", "FULL"]), seed=rng.randint(0, 2 ** 40))
    for k in ("requests", "finished", "total_output_tokens", "drafted_tokens", "submitted_tokens",
              "accepted_tokens", "wasted_draft_tokens", "false_prunes", "iterations", "overlap_iterations"):
        setattr(s, k, rng.randint(0, 10 ** 7))
    for k in metrics.MetricsSummary._FLOATS:
        setattr(s, k, rng.choice([0.0, 1.0, rng.uniform(0, 1), rng.uniform(0, 1e6), 1e-7 * rng.random(), 2.5e17]))
    s.spec_length_hist = [(k, rng.randint(0, 1000)) for k in (1, 2, 4, 8)]
    s.oracle_checked = rng.random() < 0.5
    s.oracle_ok = rng.random() < 0.5
    return s


@needs_ref
def test_metrics_jsonl_and_summary_csv_bytes_match_reference(tmp_path):
    if not hasattr(_ref(), "specref_write_summary"):
        pytest.skip("oracle/_ref built without a json.hpp (metrics.cpp left out)")
    rng = random.Random(9)
    for trial in range(40):
        s = _random_summary(rng)
        ints = np.array([s.requests, s.finished, s.total_output_tokens, s.drafted_tokens, s.submitted_tokens,
                         s.accepted_tokens, s.wasted_draft_tokens, s.false_prunes, s.iterations,
                         s.overlap_iterations], np.int64)
        dbls = np.array([getattr(s, k) for k in metrics.MetricsSummary._FLOATS], np.float64)
        hist = np.array([v for pair in s.spec_length_hist for v in pair], np.int64)
        rj, rc = tmp_path / f"r{trial}.jsonl", tmp_path / f"r{trial}.csv"
        assert _ref().specref_write_summary(str(rj).encode(), str(rc).encode(), s.mode.encode(), C.c_uint64(s.seed),
                                            ints.ctypes.data_as(C.c_void_p), dbls.ctypes.data_as(C.c_void_p),
                                            hist.ctypes.data_as(C.c_void_p), len(s.spec_length_hist),
                                            int(s.oracle_checked), int(s.oracle_ok)) == 0
        mj, mc = tmp_path / f"m{trial}.jsonl", tmp_path / f"m{trial}.csv"
        metrics.write_metrics_jsonl(mj, s)
        metrics.write_summary_csv(mc, s)
        assert mj.read_text() == rj.read_text()
        assert mc.read_text() == rc.read_text()

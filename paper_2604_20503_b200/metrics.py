"""Wire formats of the reference's serving outputs, so B200 runs are comparable file-for-file:

* trace CSV          — write_trace / ingest_trace            (workload.cpp:34-71)
* metrics JSON lines — write_metrics_jsonl (iterations, then one summary object)
                                                              (metrics.cpp:68-91)
* summary CSV        — write_summary_csv                      (metrics.cpp:93-113)
* MetricsSummary     — the summary fields                     (metrics.hpp:34-66)

The reference serialises with nlohmann::json: objects are key-sorted (std::map), compact
separators, doubles in shortest round-trip form — which is what ``json.dumps(sort_keys=True,
separators=(",", ":"))`` produces for finite values. tests/test_wire_formats.py checks every
writer byte-for-byte against the reference's own compiled writers (oracle/_ref).
"""
import json
import math
import re
from dataclasses import dataclass, field
from typing import List, Tuple


class ParseError(ValueError):
    """specsim::ParseError (errors.hpp:8-11)."""


# ------------------------------------------------------------------ trace CSV (workload.cpp)
def write_trace(path, records):
    """records: [(arrival_ms, input_len, output_len)] -> CSV with a header (workload.cpp:62-71)."""
    with open(path, "w") as f:
        f.write("arrival_ms,input_len,output_len\n")
        for a, i, o in records:
            f.write(f"{a:.3f},{int(i)},{int(o)}\n")


_NUM = r"[+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan)"
_ROW = re.compile(r"\s*(" + _NUM + r")\s*,\s*(" + _NUM + r")\s*,\s*(" + _NUM + r")\s*(\S)?", re.IGNORECASE)


def _parse_row(line):
    """sscanf(line, " %lf , %lf , %lf %c") == 3 and all fields >= 0 (workload.cpp:16-27)."""
    m = _ROW.match(line)
    if not m or m.group(4) is not None:
        return None
    a, i, o = (float(m.group(k)) for k in (1, 2, 3))
    if a < 0 or i < 0 or o < 0 or math.isnan(a) or math.isnan(i) or math.isnan(o):
        return None
    return (a, int(i), int(o))


def ingest_trace(path):
    """Parse a trace CSV (workload.cpp:34-60): blank lines skipped, an unparsable FIRST content
    line is a header, any later malformed row raises ParseError; stable-sorted by arrival."""
    try:
        f = open(path)
    except OSError as e:
        raise ParseError(f"{path}: cannot open trace file") from e
    out = []
    first = True
    with f:
        for no, line in enumerate(f.read().split("\n"), 1):
            if not line.strip():
                continue
            rec = _parse_row(line)
            if rec is None:
                if first:
                    first = False
                    continue
                raise ParseError(f"{path}:{no}: malformed trace row: {line}")
            first = False
            out.append(rec)
    out.sort(key=lambda r: r[0])  # Python's sort is stable, like std::stable_sort
    return out


# ------------------------------------------------------------------ metrics (metrics.hpp/.cpp)
@dataclass
class MetricsSummary:
    mode: str = ""
    seed: int = 0
    requests: int = 0
    finished: int = 0
    total_output_tokens: int = 0
    makespan_ms: float = 0.0
    throughput_tok_s: float = 0.0
    mean_request_latency_ms: float = 0.0
    p50_request_latency_ms: float = 0.0
    p99_request_latency_ms: float = 0.0
    mean_tpot_ms: float = 0.0
    global_tpot_ms: float = 0.0
    draft_time_ms: float = 0.0
    verify_time_ms: float = 0.0
    overhead_time_ms: float = 0.0
    verify_share: float = 0.0
    drafted_tokens: int = 0
    submitted_tokens: int = 0
    accepted_tokens: int = 0
    acceptance_ratio: float = 0.0
    wasted_draft_tokens: int = 0
    false_prunes: int = 0
    layer_work: float = 0.0
    layer_work_full: float = 0.0
    iterations: int = 0
    overlap_iterations: int = 0
    early_exit_layer_hist: List[Tuple[int, int]] = field(default_factory=list)
    spec_length_hist: List[Tuple[int, int]] = field(default_factory=list)
    batch_size_hist: List[Tuple[int, int]] = field(default_factory=list)
    oracle_checked: bool = False
    oracle_ok: bool = True

    _FLOATS = ("makespan_ms", "throughput_tok_s", "mean_request_latency_ms", "p50_request_latency_ms",
               "p99_request_latency_ms", "mean_tpot_ms", "global_tpot_ms", "draft_time_ms", "verify_time_ms",
               "overhead_time_ms", "verify_share", "acceptance_ratio", "layer_work", "layer_work_full")

    def as_json(self):
        d = {"record": "summary"}
        for k, v in self.__dict__.items():
            if k.endswith("_hist"):
                v = [[int(a), int(b)] for a, b in v]
            elif k in self._FLOATS:
                v = float(v)
            d[k] = v
        return d


def _dump(obj):
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), allow_nan=False)


def write_metrics_jsonl(path, summary: MetricsSummary, iterations=()):
    """One JSON object per iteration record (dicts with the IterationRecord fields, written
    as given plus "record": "iteration"), then the summary object (metrics.cpp:68-91)."""
    with open(path, "w") as f:
        for it in iterations:
            f.write(_dump(dict(it, record="iteration")) + "\n")
        f.write(_dump(summary.as_json()) + "\n")


_CSV_FIELDS = ("mode", "seed", "requests", "finished", "total_output_tokens", "makespan_ms", "throughput_tok_s",
               "mean_request_latency_ms", "p50_request_latency_ms", "p99_request_latency_ms", "mean_tpot_ms",
               "global_tpot_ms", "verify_share", "acceptance_ratio", "wasted_draft_tokens", "false_prunes",
               "layer_work", "layer_work_full", "oracle_ok")


def summary_csv_rows(summaries):
    """Header + one row per summary (metrics.cpp:93-113; several rows = the ablation table)."""
    lines = [",".join(_CSV_FIELDS)]
    for s in summaries:
        j = s.as_json()
        cells = []
        for k in _CSV_FIELDS:
            cell = _dump(j[k])
            cells.append(cell[1:-1] if cell.startswith('"') else cell)
        lines.append(",".join(cells))
    return "\n".join(lines) + "\n"


def write_summary_csv(path, summaries):
    if isinstance(summaries, MetricsSummary):
        summaries = [summaries]
    with open(path, "w") as f:
        f.write(summary_csv_rows(summaries))

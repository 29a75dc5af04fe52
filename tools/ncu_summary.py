"""Summarise an ncu --csv launch list: per (kernel, grid) average duration, DRAM bytes, GB/s."""
import collections
import csv
import sys


def load(fn):
    lines = [l for l in open(fn) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    idx, mv, g, mn, rid = (h.index(k) for k in ("Kernel Name", "Metric Value", "Grid Size", "Metric Name", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[r[rid]][r[mn]] = float(r[mv].replace(",", ""))
        per[r[rid]]["name"] = r[idx].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:42]
        per[r[rid]]["grid"] = r[g]
    return per


def main(fn, top=25):
    per = load(fn)
    d = collections.defaultdict(list)
    for v in per.values():
        d[(v["name"], v["grid"])].append(v)
    tot = sum(v["gpu__time_duration.sum"] for v in per.values()) / 1000
    print(f"{fn}: {len(per)} launches, {tot:.1f} us total (cold-cache, serialised)")
    for k, v in sorted(d.items(), key=lambda kv: -sum(x["gpu__time_duration.sum"] for x in kv[1]))[:top]:
        t = sum(x["gpu__time_duration.sum"] for x in v) / len(v) / 1000
        rd = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in v) / len(v) / 1e6
        share = 100 * sum(x["gpu__time_duration.sum"] for x in v) / 1000 / tot
        print(f"  {k[0]:42s} {k[1]:13s} n={len(v):4d} avg={t:8.2f}us share={share:5.1f}%  dram={rd:8.2f}MB  {rd / t if t else 0:5.2f} TB/s")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

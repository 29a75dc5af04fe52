# validation: prefill 256..511-row rule; admissions across lengths; default bench x2; GPU tests
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for L in 200 260 300 400 500 576 700 800 1000; do timeout 200 python tools/prefill_perf.py cfg3 $L 4 2>&1 | tail -1; done
for r in 1 2; do timeout 300 python bench.py > gpurun_out/bench_default_v9_$r.json 2>/dev/null; tail -1 gpurun_out/bench_default_v9_$r.json | cut -c1-160; done

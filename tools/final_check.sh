timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r01_tma.json 2> gpurun_out/bench_r01_tma.err; tail -1 gpurun_out/bench_r01_tma.json

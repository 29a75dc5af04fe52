#!/bin/bash
# round-2 GPU call 77: HEAD: full GPU suite, smoke, default bench line (driver-style 20/5 and default), reference arm
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/r77_gpu_tests.log 2>&1; echo "suite rc=$?" >> gpurun_out/r77_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r77_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r77_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r77_bench_s20.json 2> gpurun_out/r77_bench.err; echo "bench rc=$?" >> gpurun_out/r77_bench.err
timeout 1200 python bench.py > gpurun_out/r77_bench.json 2>> gpurun_out/r77_bench.err; echo "bench rc=$?" >> gpurun_out/r77_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r77_ref.json 2> gpurun_out/r77_ref.err; echo "ref rc=$?" >> gpurun_out/r77_ref.err

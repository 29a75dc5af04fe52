#!/bin/bash
# round-2 GPU call 88 (fresh container re-entry): HEAD validation — GPU suite, smoke, bench 20/5 + default, reference arm
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r88_suite.txt 2>&1; echo "suite rc=$?" >> gpurun_out/r88_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r88_suite.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r88_suite.txt
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r88_bench_s20.json 2> gpurun_out/r88_bench_s20.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r88_ref.json 2> gpurun_out/r88_ref.err

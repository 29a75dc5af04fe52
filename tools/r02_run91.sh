#!/bin/bash
# round-2 GPU call 91: sampling in EE modes (perturbed rank estimator) + temperature sweep on config 3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sampling_gpu.py tests/test_llama_gpu.py -q -x > gpurun_out/r91_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r91_tests.txt
O=gpurun_out/r91_temp_sweep.jsonl; : > $O
for t in 0 0.05 0.1 0.2 0.5 1.0; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sweep --temperature $t 2>/dev/null | tail -1 >> $O
done
for t in 0 0.1; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sweep --mode vsd_ee --gate-layer 2 --recovery --temperature $t 2>/dev/null | tail -1 >> $O
done

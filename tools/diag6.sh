cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_trace_gpu.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload cfg4 --trace 10 --batch 64 2>&1 | tail -2 > gpurun_out/trace_cfg4.json
cat gpurun_out/trace_cfg4.json

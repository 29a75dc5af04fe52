cd $GRAFT_REPO_ROOT
timeout 120 python tools/llama_perf.py tiny 4 4 2>&1 | tail -3
timeout 300 python -m pytest tests/test_llama_gpu.py -x -q 2>&1 | tail -15
timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -2
timeout 200 python tools/llama_perf.py cfg3 1 4 2>&1 | tail -2
timeout 200 python tools/llama_perf.py cfg3 64 4 2>&1 | tail -2

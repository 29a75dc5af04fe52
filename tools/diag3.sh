cd $GRAFT_REPO_ROOT
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 8 python tools/llama_perf.py tiny 2 4 2>&1 | head -80

cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for B in 1 32 128; do timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; done
timeout 300 python tools/gemm_stream.py 2560,128,2048 2048,128,2048 11264,128,2048 2048,128,5632 32000,128,2048 2304,32,768 768,32,768 6144,32,768 768,32,3072

cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_llama_gpu.py -x -q 2>&1 | tail -2
for B in 8 32 128; do echo "B=$B mt1"; FASER_ATTN_MT1=1 timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; echo "B=$B mt2"; timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; done
echo cfg4; FASER_ATTN_MT1=1 timeout 300 python tools/llama_perf.py cfg4 32 4 2>&1 | tail -1; timeout 300 python tools/llama_perf.py cfg4 32 4 2>&1 | tail -1

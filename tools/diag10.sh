cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
S="2560,128,2048 2048,128,2048 11264,128,2048 2048,128,5632 32000,128,2048 2304,32,768 768,32,768 6144,32,768 768,32,3072 32000,32,768 11264,512,2048"
echo legacy; FASER_GEMM_PLAN=legacy timeout 300 python tools/gemm_stream.py $S
echo new; timeout 300 python tools/gemm_stream.py $S
for B in 1 32 128; do echo "B=$B legacy"; FASER_GEMM_PLAN=legacy timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; echo "B=$B new"; timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; done

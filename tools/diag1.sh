set -x
cd $GRAFT_REPO_ROOT
for B in 1 32 128; do timeout 300 python tools/llama_perf.py cfg3 $B 4; done
FASER_NO_PDL=1 timeout 300 python tools/llama_perf.py cfg3 32 4
FASER_CUDA_GRAPH=1 timeout 300 python tools/llama_perf.py cfg3 32 4
timeout 300 python tools/gemm_stream.py 2560,128,2048 2048,128,2048 11264,128,2048 2048,128,5632 32000,128,2048 2304,32,768 768,32,768 6144,32,768 768,32,3072 32000,32,768 2560,4,2048 11264,4,2048
timeout 300 python tools/llama_perf.py cfg4 32 4

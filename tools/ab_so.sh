# A/B of TMA issue layouts (FASER_TMA_ISSUE) on GEMM shapes and the config-3 step
for r in 1 2; do for v in 1 4; do echo "== $v"; FASER_TMA_ISSUE=$v timeout 300 python tools/gemm_stream.py 2560,160,2048 2048,160,2048 11264,160,2048 2048,160,5632 32000,160,2048 2048,576,5632 11264,1024,2048 6144,32,768 32000,32,768 28672,64,4096; done; done
for v in 1 4; do echo "== $v"; FASER_TMA_ISSUE=$v timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; FASER_TMA_ISSUE=$v timeout 200 python tools/llama_perf.py cfg3 128 4 2>&1 | tail -1; done

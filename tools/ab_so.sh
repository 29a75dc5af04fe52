# attention two-page steps (FASER_ATTN_WIDE) : parity under the env, then A/B
FASER_ATTN_WIDE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "attn or attention or llama or trace" 2>&1 | tail -2
for r in 1 2; do for v in 0 1; do echo "== wide $v"; FASER_ATTN_WIDE=$v timeout 120 python tools/attn_bench.py 32,4,600 32,4,1200 32,4,64 128,4,600 32,1,600 1,4,600 8,4,2400; done; done
for v in 0 1; do echo "== wide $v"; FASER_ATTN_WIDE=$v timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; FASER_ATTN_WIDE=$v timeout 200 python tools/llama_perf.py cfg3 128 4 2>&1 | tail -1; done

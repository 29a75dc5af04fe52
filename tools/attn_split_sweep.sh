# split-KV CTA target sweep for the paged attention (FASER_ATTN_CTAS) at verify shapes + config-3 step
for t in 148 300 444 600 900; do echo "== $t"; FASER_ATTN_CTAS=$t timeout 120 python tools/attn_bench.py 32,4,600 32,4,1000 64,4,600 128,4,600 16,4,600 32,1,600 64,1,600; done
for t in 148 444 900; do echo "== $t"; FASER_ATTN_CTAS=$t timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; FASER_ATTN_CTAS=$t timeout 200 python tools/llama_perf.py cfg3 64 4 2>&1 | tail -1; done

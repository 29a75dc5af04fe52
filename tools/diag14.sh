cd $GRAFT_REPO_ROOT
for B in 64 128 256; do
 echo "B=$B"; PERF_STEPS=30 timeout 300 python tools/llama_perf.py cfg3 $B 4 0 2>&1 | tail -1
 for gl in 2 4; do PERF_STEPS=30 timeout 300 python tools/llama_perf.py cfg3 $B 4 2 $gl 2>&1 | tail -1; done
done

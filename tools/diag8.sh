cd $GRAFT_REPO_ROOT
for sk in 0 1 2 4 8 16 30 31; do echo "SKIP $sk"; FASER_SKIP=$sk timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; done

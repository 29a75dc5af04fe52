cd $GRAFT_REPO_ROOT
FASER_MEGA_MINB=4 FASER_MEGA_TRACE=1 timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | grep -B3 -A16 "CTA0 jobs" | head -24

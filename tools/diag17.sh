cd $GRAFT_REPO_ROOT
FASER_ATTN_MT1=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 60 -c 1 -o gpurun_out/attn_prof python tools/llama_perf.py cfg3 32 4 > gpurun_out/diag17.log 2>&1
tail -3 gpurun_out/diag17.log

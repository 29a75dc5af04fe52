cd $GRAFT_REPO_ROOT
FASER_MEGA_MINB=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mega_kernel -s 4 -c 1 -o gpurun_out/mega_prof2 python tools/llama_perf.py cfg3 32 4 > gpurun_out/diag5.log 2>&1
tail -3 gpurun_out/diag5.log

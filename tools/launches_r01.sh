cd $GRAFT_REPO_ROOT
PROFILE_ONE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/llama_perf.py cfg3 32 4 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/step_launches.csv > gpurun_out/step_launches_summary.txt

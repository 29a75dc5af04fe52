cd $GRAFT_REPO_ROOT
# one steady-state serving step (config 3, B=32), and the bench command itself (short run)
PROFILE_ONE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/llama_perf.py cfg3 32 4 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/step_launches.csv > gpurun_out/step_launches_summary.txt
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 4 --warmup 3 > gpurun_out/bench_under_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/bench_launches.csv > gpurun_out/bench_launches_summary.txt

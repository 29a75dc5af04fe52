cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
STEPS=30 timeout 1500 bash tools/sweep.sh gpurun_out/sweep.jsonl
timeout 400 python bench.py --workload cfg4 --steps 20 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt

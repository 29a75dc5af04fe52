#!/bin/bash
# round-2 GPU call 99: config 5 (70B-shape target) at TP=1 on one B200: B=32 bench line; ncu launch list of steady-state GEMMs (per-launch DRAM bytes / duration)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python bench.py --workload cfg5 --batch 32 --steps 8 --warmup 3 > gpurun_out/r99_cfg5_tp1_b32.json 2> gpurun_out/r99_cfg5_tp1_b32.err; echo "rc=$?" >> gpurun_out/r99_cfg5_tp1_b32.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_kernel --launch-skip 2400 -c 700 --csv --log-file gpurun_out/r99_cfg5_launches.csv python bench.py --workload cfg5 --batch 8 --steps 3 --warmup 3 > gpurun_out/r99_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r99_cfg5_launches.csv > gpurun_out/r99_cfg5_launches_summary.txt 2>&1
rm -f gpurun_out/r99_cfg5_launches.csv

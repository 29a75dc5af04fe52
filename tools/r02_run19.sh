#!/bin/bash
# round-2 GPU call 19: default bench line (sweep + CPU baseline) and reference arm at HEAD; ncu launch
# list of the bench command; ncu --set full of the dominant verify GEMM (128 rows) and traffic
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/r19_box.txt 2>&1
timeout 1200 python bench.py > gpurun_out/r19_bench.json 2> gpurun_out/r19_bench.err; echo "bench rc=$?" >> gpurun_out/r19_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r19_ref.json 2> gpurun_out/r19_ref.err; echo "ref rc=$?" >> gpurun_out/r19_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r19_bench_launches.csv python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/r19_bench_under_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r19_bench_launches.csv > gpurun_out/r19_bench_launches_summary.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 200 -c 4 -o gpurun_out/r19_verify_gemm python tools/layer_chain.py --rows 128 --layers 22 --reps 1 > /dev/null 2>&1

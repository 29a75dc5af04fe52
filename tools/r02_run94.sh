#!/bin/bash
# round-2 GPU call 94: HEAD validation — GPU suite + smoke, default bench, driver-style bench, reference arm, ncu launch list, memcheck of the sampling epilogue
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r94_suite.txt 2>&1; echo "suite rc=$?" >> gpurun_out/r94_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r94_suite.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r94_suite.txt
timeout 900 python bench.py > gpurun_out/r94_bench.json 2> gpurun_out/r94_bench.err
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r94_bench_s20.json 2> gpurun_out/r94_bench_s20.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r94_ref.json 2> gpurun_out/r94_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r94_bench_launches.csv python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/r94_bench_under_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r94_bench_launches.csv > gpurun_out/r94_bench_launches_summary.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_sampling_gpu.py -q -x -k "k4 and tiny-1.0 or early_exit" > gpurun_out/r94_memcheck_sampling.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/r94_memcheck_sampling.txt
rm -f gpurun_out/r94_bench_launches.csv

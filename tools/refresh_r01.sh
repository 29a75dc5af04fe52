# refresh the committed bench lines after the TMA-issue change, at the step counts of the earlier files
timeout 600 python bench.py --workload cfg4 --steps 20 > gpurun_out/r01_cfg4_bench_b32_s20_v3.json 2>/dev/null
for b in 1 8 32 64 128 256; do timeout 600 python bench.py --batch $b --steps 30 > gpurun_out/r01_cfg3_b${b}_s30_v3.json 2>/dev/null; done

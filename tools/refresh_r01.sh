# final round-1 bench lines with the current plans: batch sweep (30 steps), default bench, config 4
for b in 1 8 16 32 64 128 256; do timeout 600 python bench.py --batch $b --steps 30 2>/dev/null | tail -1; done > gpurun_out/r01_cfg3_batch_sweep_final_s30.jsonl
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/r01_bench_cfg3_final.json
timeout 600 python bench.py --workload cfg4 --steps 20 2>/dev/null | tail -1 > gpurun_out/r01_cfg4_final_s20.json
timeout 900 python bench.py --workload cfg4 2>/dev/null | tail -1 > gpurun_out/r01_cfg4_final_s60.json

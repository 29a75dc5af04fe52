#!/bin/bash
# round-2 GPU call 65: toy (config 2) step anatomy: kernel durations (ncu launch list) + bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python bench.py --workload toy --steps 200 --warmup 20 > gpurun_out/r65_toy.json 2> gpurun_out/r65_toy.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r65_toy_launches.csv python bench.py --workload toy --steps 20 --warmup 3 > /dev/null 2>&1

#!/bin/bash
# round-2 GPU call 93: functional check of bench.py's N>1 launcher path on one GPU (2 replicas share cuda:0, gloo reduction; not a perf number) + reference arm under torchrun
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
export FASER_BENCH_SHARE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 6 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/r93_n2.json 2> gpurun_out/r93_n2.err; echo "rc=$?" >> gpurun_out/r93_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r93_ref_n2.json 2> gpurun_out/r93_ref_n2.err; echo "rc=$?" >> gpurun_out/r93_ref_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --workload toy --gpus 2 --steps 6 --warmup 3 > gpurun_out/r93_toy_n2.json 2> gpurun_out/r93_toy_n2.err; echo "rc=$?" >> gpurun_out/r93_toy_n2.err

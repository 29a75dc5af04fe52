cd $GRAFT_REPO_ROOT
timeout 2700 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 4 python tools/ablate.py --workload cfg3 --seconds 1.5 --rate 220 --batch 64 --gate-layer 2 --chunk 2 --modes FULL --out gpurun_out/rep > gpurun_out/san.log 2>&1
grep -v "Host Frame" gpurun_out/san.log | head -80 > gpurun_out/san_head.log

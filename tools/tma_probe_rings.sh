# per-ring vs per-SM TMA ingest on B200 (profiles/r01_tma_probe_rings.jsonl)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu -lcuda
for cfg in "0 20 12 128 1 0" "0 20 3 128 4 0" "0 20 3 128 4 1" "0 20 12 128 1 2" "0 20 3 128 4 3" "0 20 6 128 2 3" "0 20 2 128 4 3" "2 20 3 128 4 3" "0 20 3 256 2 3" "0 148 3 128 4 3" "0 148 3 128 4 0" "2 148 3 128 4 0" "2 148 3 128 4 3"; do timeout 60 /tmp/tma_probe $cfg; done

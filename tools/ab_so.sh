# in-stream verify-plan search for the config-3 shapes at 257..512 rows (B=128, k=4 -> 512 rows; B=96 -> 384)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 200 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
run "" 128
for c in 128,1,2 128,1,4 256,1,2 64,1,2; do run "2048,5632,257,512,$c" 128; done
for c in 128,1,1 64,1,2 128,1,2; do run "2560,2048,257,512,$c" 128; done
for c in 128,1,1 64,1,2 128,1,2; do run "2048,2048,257,512,$c" 128; done
for c in 256,2,1 128,2,1; do run "11264,2048,257,512,$c" 128; done
run "" 96
for c in 128,1,2 128,1,4; do run "2048,5632,257,512,$c" 96; done

# in-stream verify-plan search for config-3 shapes at 33..64 rows (B=16) and 1..32 rows (B=8)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
run "" 16
for c in 64,1,4 32,1,8 64,1,2; do run "2048,5632,33,64,$c" 16; done
for c in 64,1,4 32,1,2; do run "2560,2048,33,64,$c" 16; done
for c in 64,1,4 32,1,2; do run "2048,2048,33,64,$c" 16; done
for c in 64,2,1 32,1,1; do run "11264,2048,33,64,$c" 16; done
run "" 8
for c in 32,1,8 32,1,2; do run "2048,5632,1,32,$c" 8; done
for c in 32,1,2 32,1,8; do run "2048,2048,1,32,$c" 8; done
for c in 32,1,1 32,2,1; do run "11264,2048,1,32,$c" 8; done

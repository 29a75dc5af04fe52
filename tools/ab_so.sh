# in-stream validation of combined qkv + gate/up plans at 769..1024 rows
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
C="2560,2048,769,1024,128,1,1;11264,2048,769,1024,256,1,1"
for B in 256 224 200; do run "" $B; run "$C" $B; run "2560,2048,769,1024,128,1,1" $B; done
run "11264,2048,769,1024,256,1,1" 200

# wave-aware variants at 257..448 rows (B=96 -> 384 rows, B=80 -> 320)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
for B in 96 80; do
run "" $B
run "11264,2048,257,448,128,1,1,0" $B
run "11264,2048,257,448,256,1,1,0" $B
run "2048,2048,257,448,32,1,1,0" $B
run "2048,2048,257,448,64,1,1,1" $B
run "2560,2048,257,448,64,1,1,0" $B
done

# wave-aware shallow variants at 129..224 rows (B=40 -> 160, B=48 -> 192, B=56 -> 224)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
for B in 48 40 56; do
run "" $B
run "11264,2048,129,224,128,1,1,0" $B
run "2560,2048,129,224,32,1,1,0" $B
run "2560,2048,129,224,64,1,1,0" $B
run "2048,2048,129,224,32,1,1,0" $B
done

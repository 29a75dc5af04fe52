# in-stream verify-plan search for config-3 shapes at 513..768 rows (B=160 -> 640 rows, B=192 -> 768)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
for B in 160 192; do
run "" $B
run "2048,5632,513,768,128,1,1" $B
run "2048,5632,513,768,128,1,2" $B
run "2048,2048,513,768,128,1,1" $B
run "2560,2048,513,768,128,1,1" $B
run "11264,2048,513,768,256,1,1" $B
run "11264,2048,513,768,256,2,1" $B
done

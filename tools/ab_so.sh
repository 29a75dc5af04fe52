# prefill gate/up just above 256 rows (bn 256 leaves a nearly empty second token tile)
run() { echo "== L=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 200 python tools/prefill_perf.py cfg3 $2 4 2>&1 | tail -1; }
for L in 260 300 350; do run "" $L; run "11264,2048,257,400,128,2,1" $L; run "11264,2048,257,400,256,2,1" $L; run "11264,2048,257,400,128,1,1" $L; done

# in-stream verify-plan A/B for the config-3 down GEMM (2048x5632) at 65..128 rows
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; }
for r in 1 2; do
run ""
run "2048,5632,65,128,64,1,4"
run "2048,5632,65,128,64,1,3"
run "2048,5632,65,128,64,1,6"
run "2048,5632,65,128,64,2,4"
run "2048,5632,65,128,32,1,4"
done

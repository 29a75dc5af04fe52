# in-stream prefill plan A/B (FASER_PLAN_OVERRIDE) on a 576-token admission (tools/prefill_perf.py)
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 200 python tools/prefill_perf.py cfg3 576 6 2>&1 | tail -1; }
run ""
run "2048,5632,256,1023,128,1,1"
run "2048,5632,256,1023,64,1,2"
run "2048,5632,256,1023,256,1,4"
run "2048,5632,256,1023,64,2,2"
run "2048,2048,256,1023,128,1,1"
run "2048,2048,256,1023,64,1,2"
run "2560,2048,256,1023,64,1,1"
run "2560,2048,256,1023,64,2,1"
run ""

# shallow (2 CTAs/SM) variants at 129..256 rows (B=64)
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 64 4 2>&1 | tail -1; }
run ""
for c in 128,1,1,0 64,1,1,0 128,1,2,0; do run "11264,2048,129,256,$c"; done
run "2560,2048,241,256,32,1,1,0"
run "2048,2048,129,256,32,1,1,0"
run "2048,2048,129,256,64,1,1,0"
run ""

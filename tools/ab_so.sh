# shallow draft-plan variants at 33..64 rows (B=64 draft steps)
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 64 4 2>&1 | tail -1; }
run ""
for c in 32,1,1,0 32,1,2,0 64,1,2,0; do run "6144,768,33,64,$c"; done
for c in 32,1,2,0 32,1,4,0 64,1,4,0; do run "2304,768,33,64,$c"; done
for c in 32,1,4,0 64,1,4,1; do run "768,3072,33,64,$c"; done
run ""

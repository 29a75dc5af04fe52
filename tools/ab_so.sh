# shallow draft-plan variants at 17..32 rows (B=32 draft steps)
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; }
run ""
for c in 32,1,1,0 32,1,2,0 32,1,3,0; do run "6144,768,17,32,$c"; done
for c in 32,1,3,0 32,1,2,0; do run "2304,768,17,32,$c"; done
run "768,768,17,32,32,1,3,0"
run ""

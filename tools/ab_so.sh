# in-stream draft-plan search for the config-4 draft shapes at 17..32 rows (B=32)
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 300 python tools/llama_perf.py cfg4 32 4 2>&1 | tail -1; }
run ""
for c in 32,2,1 32,1,2 64,1,1; do run "16384,2048,17,32,$c"; done
for c in 32,1,4 64,1,4 32,1,2; do run "3072,2048,17,32,$c"; done
for c in 32,1,2 32,1,8; do run "2048,2048,17,32,$c"; done
for c in 32,2,1 64,4,1; do run "128256,2048,17,32,$c"; done

# shallow (2 CTAs/SM) vs deep plans for the under-filled config-3 gate/up at 65..128 rows (B=32)
run() { echo "== $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; }
run ""
for c in 128,1,2,0 128,1,3,0 64,1,1,0 64,1,2,0 128,1,1,0; do run "11264,2048,65,128,$c"; done
for c in 128,1,2,0 64,1,1,0; do run "32000,2048,65,128,$c"; done
run "2048,5632,65,128,64,1,4,0"

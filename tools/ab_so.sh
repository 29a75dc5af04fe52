# in-stream draft-plan search (config-3 draft shapes) at 97..128 rows (B=128) and 193..256 rows (B=256)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
run "" 128
for c in 64,1,1 128,1,1 64,1,2; do run "2304,768,97,128,$c" 128; done
for c in 64,1,1 128,1,1 128,2,1; do run "6144,768,97,128,$c" 128; done
for c in 64,1,4 128,1,4 128,1,2; do run "768,3072,97,128,$c" 128; done
for c in 64,1,1 128,1,3; do run "768,768,97,128,$c" 128; done
run "" 256
for c in 128,1,1 64,1,2 256,1,1; do run "2304,768,193,256,$c" 256; done
for c in 128,1,1 128,2,1 256,1,1; do run "6144,768,193,256,$c" 256; done
for c in 64,1,2 128,1,2 128,1,4; do run "768,3072,193,256,$c" 256; done
for c in 64,1,2 128,1,2; do run "768,768,193,256,$c" 256; done

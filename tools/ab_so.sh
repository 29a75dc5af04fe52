# shallow (2 CTAs/SM) variants at 449..512 rows (B=128) and 769..1024 rows (B=256)
run() { echo "== B=$2 $1"; FASER_PLAN_OVERRIDE="$1" timeout 250 python tools/llama_perf.py cfg3 $2 4 2>&1 | tail -1; }
run "" 128
run "2560,2048,449,512,64,1,1,0" 128
run "11264,2048,449,512,256,1,1,0" 128
run "11264,2048,449,512,128,1,1,0" 128
run "2048,2048,449,512,64,1,1,0" 128
run "" 256
run "11264,2048,769,1024,256,1,1,0" 256
run "2560,2048,769,1024,128,1,1,0" 256

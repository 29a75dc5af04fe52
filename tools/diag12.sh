cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for B in 1 32 128; do echo "B=$B legacy"; FASER_GEMM_PLAN=legacy timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; echo "B=$B new"; timeout 200 python tools/llama_perf.py cfg3 $B 4 2>&1 | tail -1; done
for B in 128 256; do
 echo "== B=$B vsd"; timeout 300 python bench.py --batch $B --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p50_tpot_ms'], d['acceptance'], d['ms_per_step'])"
 for gl in 2 4; do echo "== B=$B ee gate $gl"; timeout 300 python bench.py --batch $B --steps 30 --mode ee --gate-layer $gl --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p50_tpot_ms'], d['acceptance'], d['ms_per_step'], d.get('layer_work_per_drafted_token'))"; done
 echo "== B=$B ov chunk2"; timeout 300 python bench.py --batch $B --steps 30 --mode ov --chunk 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p50_tpot_ms'], d['acceptance'], d['ms_per_step'])"
done

cd $GRAFT_REPO_ROOT
for B in 128 256; do
 for gl in 2 8; do echo "== B=$B vsd_ee gate $gl"; timeout 300 python bench.py --batch $B --steps 30 --mode vsd_ee --gate-layer $gl --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p50_tpot_ms'], d['acceptance'], d['ms_per_step'], d.get('layer_work_per_drafted_token'), d['device_ms_per_step'])"; done
 echo "== B=$B vsd"; timeout 300 python bench.py --batch $B --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['p50_tpot_ms'], d['acceptance'], d['ms_per_step'], d['device_ms_per_step'])"
done

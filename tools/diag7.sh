cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --workload tp_tiny --tp --steps 5 --warmup 3 --batch 8 2>&1 | tail -2

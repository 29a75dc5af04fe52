# A/B of product-library builds (ab_old.so / ab_new.so at the repo root, untracked): PDL-launched attention
L=paper_2604_20503_b200/libfaser_b200.so
cp ab_new.so $L; timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do for v in old new; do cp ab_$v.so $L; echo "== $v"; timeout 200 python tools/llama_perf.py cfg3 32 4 2>&1 | tail -1; timeout 200 python tools/llama_perf.py cfg3 128 4 2>&1 | tail -1; timeout 300 python tools/llama_perf.py cfg4 32 4 2>&1 | tail -1; done; done
cp ab_new.so $L

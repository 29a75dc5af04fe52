#!/bin/bash
# round-2 GPU call 100 (re-run as 102 after the TP vocab padding): final HEAD GPU suite + smoke
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r100_suite.txt 2>&1; echo "suite rc=$?" >> gpurun_out/r100_suite.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r100_suite.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r100_suite.txt

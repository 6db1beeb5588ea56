#!/bin/bash
# panel change check: microbench, numeric GPU tests, C3 orthogonality, C4/C3 bench lines
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/${TAG:-pc}
timeout 120 tools/bench_panel > $O.panel.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O.pytest.log 2>&1; echo "pytest exit $?" >> $O.pytest.log
SKIP_CUSOLVER=1 SIZES=16384 timeout 300 python tools/orth_accurate.py > $O.orth.json 2>/dev/null
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O.c4.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $O.c3.json 2>/dev/null
echo done

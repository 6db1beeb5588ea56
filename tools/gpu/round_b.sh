#!/bin/bash
# new GPU tests (nb=128, padding, Asap/GrASAP at scale), thesis grid, Asap/GrASAP bench lines
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_numeric_gpu.py -x -q -k "nb128 or padded or asap_grasap_at_scale" > gpurun_out/rb.pytest.log 2>&1; echo "exit $?" >> gpurun_out/rb.pytest.log
timeout 600 python tools/thesis_grid.py > gpurun_out/thesis_grid.json 2> gpurun_out/thesis_grid.err
for t in asap grasap; do
  timeout 300 python bench.py --tree $t --no-cpu-baseline --no-e2e > gpurun_out/rb.c3_$t.json 2>/dev/null
done
echo done

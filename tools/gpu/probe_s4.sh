#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in "" _s4 _s6 _s9; do
timeout 60 ./tools/bench_panel$v > gpurun_out/bp$v.txt 2>&1; echo "exit $?" >> gpurun_out/bp$v.txt
done
timeout 600 python -m pytest tests/test_numeric_gpu.py -m gpu -x -q > gpurun_out/la.pytest.log 2>&1; echo "exit $?" >> gpurun_out/la.pytest.log
for c in c4 c3 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/la.$c.json 2>gpurun_out/la.$c.err
done
echo done

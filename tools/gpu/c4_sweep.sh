#!/bin/bash
# C4 panel-weight sweep under the plan's dequeue policy
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for w in 4 6 8 12 20; do
  TQR_COST_PANEL=$w timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/c4w_$w.json 2>/dev/null
done
echo done

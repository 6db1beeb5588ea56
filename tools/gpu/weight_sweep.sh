#!/bin/bash
# panel-weight sweep of the list schedule on the throughput-bound configs
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for w in 2 3 4 6; do
  TQR_COST_PANEL=$w timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/c3w_$w.json 2>/dev/null
  TQR_COST_PANEL=$w timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/c5w_$w.json 2>/dev/null
done
echo done

#!/bin/bash
# priority panel-weight sweep of the list schedule (panels simulated at weight 8) on C3 (resident + e2e) and C5
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for w in 2 3 4 6 8; do
  TQR_COST_PANEL=$w timeout 400 python bench.py --config c3 --no-cpu-baseline --steps 3 > gpurun_out/c3w_$w.json 2>/dev/null
  TQR_COST_PANEL=$w timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/c5w_$w.json 2>/dev/null
done
echo done

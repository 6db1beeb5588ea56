#!/bin/bash
# panel list-schedule weight sweep on C3 and the C5 shard (throughput-bound schedules)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for w in 2 3 4 5; do
  TQR_COST_PANEL=$w timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/w_c3_$w.json 2>/dev/null
done
for w in 2 3 4 5; do
  TQR_COST_PANEL=$w timeout 600 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/w_c5_$w.json 2>/dev/null
done
echo done

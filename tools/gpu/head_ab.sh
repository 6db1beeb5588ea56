#!/bin/bash
# C3 head/tail: timelines with the current executor, simulated panel length 1 vs 2.8
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for s in 1 2.8; do
  TQR_SIM_PANEL=$s timeout 600 python tools/item_trace.py --config c3 --out gpurun_out/head_$s.json --gantt gpurun_out/head_$s.csv > /dev/null 2>&1
  gzip -f gpurun_out/head_$s.csv
done
echo done

#!/bin/bash
# Sweep of the list-schedule panel weight (TQR_COST_PANEL) on C4 and C3 bench lines -> gpurun_out/sweep.log
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in 4 6 8 10 14 20 30; do echo "c4 panel=$c $(TQR_COST_PANEL=$c timeout 120 python bench.py --config c4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["ms_per_step"], d["kernel_ms_each"])')" >> gpurun_out/sweep.log; done
for c in 2 2.5 3 4 5; do echo "c3 panel=$c $(TQR_COST_PANEL=$c timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["ms_per_step"], d["kernel_ms_each"])')" >> gpurun_out/sweep.log; done

#!/bin/bash
# (pre-session-4 semantics: TQR_SIM_PANEL was a multiplier; it is now an absolute weight)
# C4 sweep of the simulated panel duration (TQR_SIM_PANEL, multiplier of the
# panel weight in the list-schedule simulation) at the default priority weight
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for m in 0.6 0.8 1.0 1.25 1.5 2.0; do echo "c4 sim_panel=$m $(TQR_SIM_PANEL=$m timeout 120 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 8 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["ms_per_step"], d["kernel_ms_each"])')" >> gpurun_out/sweep2.log; done
for w in 7 8 9; do echo "c4 panel=$w $(TQR_COST_PANEL=$w timeout 120 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 8 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["ms_per_step"])')" >> gpurun_out/sweep2.log; done

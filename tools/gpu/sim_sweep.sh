#!/bin/bash
# (pre-session-4 semantics: TQR_SIM_PANEL was a multiplier; it is now an absolute weight)
# C3: simulated panel duration (TQR_SIM_PANEL x priority weight) sweep
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for s in 1 1.5 2 2.8; do
  TQR_SIM_PANEL=$s timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/sim_c3_$s.json 2>/dev/null
done
for s in 1 2.8; do
  TQR_SIM_PANEL=$s TQR_FLAGS=4 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/sim_c3_$s.f4.json 2>/dev/null
done
echo done

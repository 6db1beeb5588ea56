#!/bin/bash
# e2e sensitivity to the modeled H2D rate (TQR_H2D_GBS) and the simulated panel weight (TQR_SIM_PANEL,
# absolute, in update-slab units; default 8) of the arrival-aware list schedule
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 900 python bench.py "$@" --no-cpu-baseline --steps 3 > gpurun_out/e2e_$tag.json 2>/dev/null; }
run c3 TQR_DUMMY=1
run c3old TQR_SIM_PANEL=1 TQR_H2D_GBS=48
run c4 TQR_DUMMY=1 --config c4
run c5 TQR_DUMMY=1 --config c5
run c5old TQR_SIM_PANEL=1 TQR_H2D_GBS=48 --config c5
echo done

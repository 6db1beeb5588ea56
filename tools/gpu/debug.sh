#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/debug_scaled.py > gpurun_out/debug.log 2>&1
for b in tools/bench_panel tools/bench_panel_l2 tools/bench_panel_fast tools/bench_panel_fastl2; do echo "== $b" >> gpurun_out/debug.log; timeout 120 $b >> gpurun_out/debug.log 2>&1; done
echo done

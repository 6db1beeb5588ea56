#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/debug_tiny3.py > gpurun_out/debug2.log; timeout 120 tools/bench_panel >> gpurun_out/debug2.log 2>&1
echo done

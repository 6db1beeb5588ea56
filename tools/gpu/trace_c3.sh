#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python tools/item_trace.py --config c3 --out gpurun_out/trace_c3b.json --gantt gpurun_out/gantt_c3.csv > gpurun_out/trace_c3b.log 2>&1
gzip -f gpurun_out/gantt_c3.csv
echo done

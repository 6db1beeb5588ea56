#!/bin/bash
# per-item device timelines (tools/item_trace.py) for C3, C4, C5 (1 GPU)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in c4 c3 c5; do
  timeout 900 python tools/item_trace.py --config $c --out gpurun_out/trace_$c.json > gpurun_out/trace_$c.log 2>&1
done
echo done

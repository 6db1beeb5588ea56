#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python tools/item_trace.py --config c3 --stream --out gpurun_out/s4.trace_c3_stream.json > gpurun_out/s4.trace_c3_stream.log 2>&1
timeout 600 python tools/item_trace.py --config c3 --out gpurun_out/s4.trace_c3.json > gpurun_out/s4.trace_c3.log 2>&1
timeout 600 python tools/item_trace.py --config c5 --out gpurun_out/s4.trace_c5.json > gpurun_out/s4.trace_c5.log 2>&1
timeout 600 python tools/item_trace.py --config c4 --out gpurun_out/s4.trace_c4.json > gpurun_out/s4.trace_c4.log 2>&1
echo done

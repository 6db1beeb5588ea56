#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/s4.c3tt.json 2>gpurun_out/s4.c3tt.err
timeout 600 python bench.py --family TS --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/s4.c3ts.json 2>gpurun_out/s4.c3ts.err
timeout 600 python bench.py --config c4 --family TS --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/s4.c4ts.json 2>gpurun_out/s4.c4ts.err
timeout 600 python tools/item_trace.py --config c3 --family TS --out gpurun_out/s4.trace_c3ts.json > gpurun_out/s4.trace_c3ts.log 2>&1
echo done

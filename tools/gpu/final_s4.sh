#!/bin/bash
# Round-end measurement (session 4): final_round.sh + ncu captures + C5 scaling probe
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
bash tools/gpu/final_round.sh ${1:-fin}
bash tools/gpu/ncu_round.sh ${1:-fin}ncu
timeout 1200 python tools/c5_scaling_probe.py > gpurun_out/${1:-fin}.c5probe.json 2> gpurun_out/${1:-fin}.c5probe.err
timeout 600 python tools/item_trace.py --config c3 --out gpurun_out/${1:-fin}.trace_c3.json > /dev/null 2>&1
timeout 600 python tools/item_trace.py --config c4 --out gpurun_out/${1:-fin}.trace_c4.json > /dev/null 2>&1
timeout 600 python tools/item_trace.py --config c5 --out gpurun_out/${1:-fin}.trace_c5.json > /dev/null 2>&1
echo all done

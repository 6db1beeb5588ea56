#!/bin/bash
# ncu captures (round 2): C3 executor, update + panel microbenchmarks, launch list
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${1:-ncu2}
NCU="ncu --set full --clock-control none --import-source on"
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$T.c3plain.json 2>&1 &&
timeout 1500 $NCU -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/$T.c3 -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$T.c3.log 2>&1
timeout 600 $NCU -k regex:k_upd -c 2 -o gpurun_out/$T.upd -f tools/bench_update > gpurun_out/$T.upd.log 2>&1
timeout 600 $NCU -k regex:k_pan -c 2 -o gpurun_out/$T.pan -f tools/bench_panel > gpurun_out/$T.pan.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$T.launches_c3.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$T.launch.log 2>&1
echo done

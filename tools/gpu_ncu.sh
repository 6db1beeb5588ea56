#!/bin/bash
# ncu --set full captures for the kernel-choice evidence (one GPU, one
# launch each): the C3 executor (nb=256), the C1 executor (nb=64 tiles), the
# update-item and panel-item microbenchmarks.  Reports in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${TAG:-ncu}
NCU="ncu --set full --clock-control none --import-source on"
# C3: warm-up launches of exec_kernel are skipped (-s 3), one captured
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$T.c3plain.json 2>&1 &&
timeout 1500 $NCU -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/$T.c3 -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$T.c3.log 2>&1
timeout 300 $NCU -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/$T.c1 -f \
  python bench.py --config c1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/$T.c1.log 2>&1
timeout 600 $NCU -k regex:k_upd -c 2 -o gpurun_out/$T.upd -f tools/bench_update > gpurun_out/$T.upd.log 2>&1
timeout 600 $NCU -k regex:k_pan -c 5 -o gpurun_out/$T.pan -f tools/bench_panel > gpurun_out/$T.pan.log 2>&1
echo done

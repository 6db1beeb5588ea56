#!/bin/bash
# panel microbenchmarks (product + instrumented level-2), outputs in gpurun_out/
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/${TAG:-panel}
for b in tools/bench_panel tools/bench_panel_*; do
  case $b in *.cu|*.sh) continue;; esac
  echo "== $b" >> $O.log; timeout 120 $b >> $O.log 2>&1
done
echo done

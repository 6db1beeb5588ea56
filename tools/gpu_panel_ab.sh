#!/bin/bash
# Panel A/B on one GPU: parity tests for the panel numerics, microbenchmarks
# of the product and the variants built by tools/build_panel_bench.sh, then
# C3/C4 bench lines and the C5 scaling projection (outputs in gpurun_out/).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
O=gpurun_out/${TAG:-ab}
timeout 900 python -m pytest tests -m gpu -x -q > $O.pytest.log 2>&1; echo "pytest exit $?" >> $O.pytest.log
for b in tools/bench_panel tools/bench_panel_*; do
  case $b in *.cu|*.sh) continue;; esac
  echo "== $b" >> $O.panel.log; timeout 120 $b >> $O.panel.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O.c3.json 2> $O.c3.err
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e > $O.c4.json 2> $O.c4.err
[ -n "$PROBE_C5" ] && timeout 900 python tools/c5_scaling_probe.py > $O.c5probe.json 2> $O.c5probe.err
echo done

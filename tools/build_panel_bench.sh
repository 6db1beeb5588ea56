#!/bin/bash
# Build the panel microbenchmark variants: tools/bench_panel (product code),
# tools/bench_panel_l2 (level-2 per-phase cycle counters), and any extra
# variant given as NAME=FLAGS arguments (e.g. serial=-DTQR_L2_SERIAL_SCALARS).
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include"
nvcc $F -o tools/bench_panel tools/bench_panel.cu &
nvcc $F -o tools/bench_update tools/bench_update.cu &
nvcc $F -DTQR_PROF_L2 -o tools/bench_panel_l2 tools/bench_panel.cu &
for v in "$@"; do
  nvcc $F ${v#*=} -o tools/bench_panel_${v%%=*} tools/bench_panel.cu &
done
wait

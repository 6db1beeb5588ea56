#!/bin/bash
# in-executor A/B of library variants (libtqr.so = product; libtqr_v*.so = ablations)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in "" _v1 _v2 _v3; do
  [ -f paper_1303_3182_b200/libtqr$v.so ] || continue
  for c in c3 c5; do
    TQR_LIB_PATH=$PWD/paper_1303_3182_b200/libtqr$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/ab$v.$c.json 2>/dev/null
  done
done
echo done

#!/bin/bash
# A/B of executor flags on C4 / C3 / C5 (TQR_FLAGS=4: no look-ahead dequeue)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for f in 0 4; do
  for c in c4 c3; do
    TQR_FLAGS=$f timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_f$f.json 2>/dev/null
  done
done
echo done

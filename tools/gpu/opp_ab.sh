#!/bin/bash
# opportunistic order A/B (TQR_FLAGS=8 disables it) + the executor determinism tests
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_numeric_gpu.py -q -x -k "deterministic or nb128 or vs_replay" > gpurun_out/opp.pytest.log 2>&1; echo "exit $?" >> gpurun_out/opp.pytest.log
for f in 0 8; do
  TQR_FLAGS=$f timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/opp_c3_$f.json 2>/dev/null
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/opp_c3_policy.json 2>/dev/null
timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/opp_c4_policy.json 2>/dev/null
TQR_FLAGS=0 timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/opp_c4_0.json 2>/dev/null
timeout 900 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/opp_c5_policy.json 2>/dev/null
echo done

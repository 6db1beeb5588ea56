#!/bin/bash
# C5: distributed-path GPU tests (binary + gather merges), scaling projection probe
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist.py -m gpu -x -q > gpurun_out/c5.pytest.log 2>&1; echo "exit $?" >> gpurun_out/c5.pytest.log
timeout 1200 python tools/c5_scaling_probe.py > gpurun_out/c5probe.json 2> gpurun_out/c5probe.err
echo done

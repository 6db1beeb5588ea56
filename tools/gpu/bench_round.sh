#!/bin/bash
# bench lines (C3 default with e2e + cpu_baseline, reference arm, C4, C5 1 GPU) + the C5 tests
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nproc; free -g | head -2
( time timeout 900 python bench.py ) > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
( time timeout 600 python bench.py --impl reference ) > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err
timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err
timeout 900 python -m pytest tests/test_c5_gpu.py -q -s > gpurun_out/c5tests.log 2>&1; echo "exit $?" >> gpurun_out/c5tests.log
echo done

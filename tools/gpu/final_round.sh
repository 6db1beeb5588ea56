#!/bin/bash
# Round-end measurement: full GPU tests, smoke, bench lines (C3 default with CPU baselines,
# reference arm, C4, C5 1 GPU, Asap/GrASAP at C3), launch list.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${1:-fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$T.gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$T.pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/$T.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T.smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/$T.smoke.log
timeout 900 python bench.py > gpurun_out/$T.c3.json 2> gpurun_out/$T.c3.err
timeout 600 python bench.py --impl reference > gpurun_out/$T.ref.json 2> gpurun_out/$T.ref.err
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/$T.c4.json 2> gpurun_out/$T.c4.err
timeout 900 python bench.py --config c5 > gpurun_out/$T.c5.json 2> gpurun_out/$T.c5.err
timeout 300 python bench.py --tree asap --no-cpu-baseline --no-e2e > gpurun_out/$T.c3asap.json 2>/dev/null
timeout 300 python bench.py --tree grasap --no-cpu-baseline --no-e2e > gpurun_out/$T.c3grasap.json 2>/dev/null
echo done

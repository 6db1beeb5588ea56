#!/bin/bash
# One-GPU round check: tests, smoke, bench lines for C3/C4/C5 + reference arm, ncu launch list (outputs in gpurun_out/).
set -x
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1

timeout 600 python tools/item_trace.py --config c3 --out gpurun_out/item_trace_c3.json > gpurun_out/item_trace_c3.log 2>&1
timeout 300 python tools/item_trace.py --config c4 --out gpurun_out/item_trace_c4.json > gpurun_out/item_trace_c4.log 2>&1
[ -n "$WITH_C5_PROBE" ] && timeout 900 python tools/c5_scaling_probe.py > gpurun_out/c5probe.json 2> gpurun_out/c5probe.err
[ -n "$WITH_NCU_FULL" ] && TAG=ncuF bash tools/gpu_ncu.sh
echo all done

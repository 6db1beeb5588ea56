#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
./tools/bench_update > gpurun_out/bu_base.txt 2>&1
./tools/bu_g1lds64 > gpurun_out/bu_g1lds64.txt 2>&1
echo done

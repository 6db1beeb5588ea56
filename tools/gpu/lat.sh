#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
./tools/fp64_lat > gpurun_out/fp64_lat.json 2>&1
echo done

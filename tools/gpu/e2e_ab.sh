#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python tools/e2e_ab.py > gpurun_out/e2e_ab.log 2>&1
echo done

#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python tools/policy_ab.py > gpurun_out/policy_ab.log 2>&1
echo done

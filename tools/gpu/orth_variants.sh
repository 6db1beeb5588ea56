#!/bin/bash
# orthogonality at C3 for libtqr variants (tqr_orth_variants): product, plain Gram, dlarfg tau
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for v in "" _plain _dlarfg; do
  TQR_LIB_PATH=paper_1303_3182_b200/libtqr$v.so SKIP_CUSOLVER=1 SIZES=16384 timeout 300 python tools/orth_accurate.py > gpurun_out/orth$v.json 2>/dev/null
done
TQR_LIB_PATH=paper_1303_3182_b200/libtqr_plain.so timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/c4_plain.json 2>/dev/null
echo done

#!/bin/bash
# In-executor A/B of kernel variants: bench lines for the product library and every
# paper_1303_3182_b200/libtqr_v*.so built with ablation macros, e.g.
#   TQR_EXTRA_NVCC_FLAGS="-DTQR_NO_DIRECT_ACC" TQR_BUILD_DIR=$PWD/build_v1 \
#   TQR_LIB_OUT=$PWD/paper_1303_3182_b200/libtqr_v1.so python -c "from paper_1303_3182_b200 import _build; _build.build()"
# (isolated-item microbenchmarks mispredicted the sign of several changes; decide on these numbers)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for lib in paper_1303_3182_b200/libtqr.so paper_1303_3182_b200/libtqr_v*.so; do
  [ -f "$lib" ] || continue
  v=$(basename "$lib" .so)
  for c in ${CONFIGS:-c3 c4 c5}; do
    TQR_LIB_PATH=$PWD/$lib timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/ab.$v.$c.json 2>/dev/null
  done
done
echo done

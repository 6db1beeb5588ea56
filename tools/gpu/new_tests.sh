cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
free -g | head -2
timeout 1500 python -m pytest tests/test_c5_gpu.py "tests/test_numeric_gpu.py::test_c3_shape_residual_orthogonality" "tests/test_numeric_gpu.py::test_tiled_qr_with_reference_elimination_list" -x -q -s --durations=10 > gpurun_out/pytest_new.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_new.log

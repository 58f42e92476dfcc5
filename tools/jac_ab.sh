#!/bin/bash
# A/B of Jacobi variants on configs[2]: parity tests with the default library, then fine-sweep timing of
# the default build, the residual form (TK_JACOBI_RESIDUAL_FORM=1) and the named variants (lib_<v>.so)
timeout 900 python -m pytest tests/test_gpu_sizes.py tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_shapes.py tests/test_slabs_gpu.py -x -q > gpurun_out/j_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/j_tests.log
TK_JACOBI_RESIDUAL_FORM=1 timeout 300 python tools/time_jacobi.py 2 resid 2>&1 | tail -1
bash tools/variant_time.sh "$@"

set -x
timeout 300 python tools/debug_ama_linf.py 0 > gpurun_out/r2d_debug_linf.log 2>&1; echo dbg rc=$?
timeout 300 python tools/debug_ama_linf.py 1 > gpurun_out/r2d_debug_l1.log 2>&1; echo dbg rc=$?
timeout 900 python -m pytest tests/test_linalg_gpu.py tests/test_cpp_mirror.py -q -rf > gpurun_out/r2d_pytest.log 2>&1; echo pytest rc=$?

set -x
make -s -C tests/cpp
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/r2f_pytest.log 2>&1; echo pytest rc=$?
timeout 2400 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 99 --print-limit 50 \
  python -m pytest tests/test_gpu_parity.py tests/test_linalg_gpu.py -m gpu -q -x -p no:cacheprovider \
  -k "not c1_exact and not test_partitioned and not ring_wraps" > gpurun_out/r2f_memcheck.log 2>&1; echo memcheck rc=$?

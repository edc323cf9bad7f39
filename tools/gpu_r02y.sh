set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "mask_path or wide_rows or c4s or hessian" > gpurun_out/r2y_pytest.log 2>&1; echo rc=$?
timeout 600 python tools/profile_gamma.py c4inf 0 1 gpurun_out/r2y_c4inf_new.json > gpurun_out/r2y_c4inf_new.log 2>&1
CPB_NO_HESS_BLK=1 timeout 600 python tools/profile_gamma.py c4inf 0 1 gpurun_out/r2y_c4inf_old.json > gpurun_out/r2y_c4inf_old.log 2>&1
timeout 900 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2y_c4_new.json 2>/dev/null
CPB_NO_HESS_BLK=1 timeout 900 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2y_c4_old.json 2>/dev/null

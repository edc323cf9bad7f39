set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mask_path or wide_rows" > gpurun_out/r2z_pytest.log 2>&1; echo rc=$?
timeout 300 python tools/profile_gamma.py c4inf 0 1 gpurun_out/r2z_c4inf_new.json > gpurun_out/r2z_c4inf_new.log 2>&1
CPB_TRACE=1 timeout 400 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r2z_c4_new.json 2>gpurun_out/r2z_c4_new.err
echo done

set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "hessian or ssnal or golden or c3 or c2 or path" > gpurun_out/r2x_pytest.log 2>&1; echo rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2x_c3_new_$i.json 2>gpurun_out/r2x_c3_new_$i.err
CPB_NO_PHI_GRAD=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2x_c3_old_$i.json 2>/dev/null
done
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2x_c2_new.json 2>/dev/null
CPB_NO_PHI_GRAD=1 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2x_c2_old.json 2>/dev/null

set -x
CPB_HESS_SLICED=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hessian or ssnal_iteration" > gpurun_out/r2w_pytest.log 2>&1; echo rc=$?
for i in 1 2; do
CPB_HESS_SLICED=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_c3_s1_$i.json 2>/dev/null
CPB_HESS_SLICED=2 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_c3_s2_$i.json 2>/dev/null
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_c3_base_$i.json 2>/dev/null
done
CPB_HESS_SLICED=1 timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_c2_s1.json 2>/dev/null
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2w_c2_base.json 2>/dev/null

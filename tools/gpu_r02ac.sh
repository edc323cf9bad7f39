set -x
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "hessian or ssnal or golden or c3 or c2" > gpurun_out/r2ac_pytest.log 2>&1; echo rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ac_c3_new_$i.json 2>/dev/null
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ac_c2_new_$i.json 2>/dev/null
done
cp abtmp/hess_tma_full.cu paper_2501_15964_b200/csrc/hess_tma.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ac_c3_old_$i.json 2>/dev/null
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ac_c2_old_$i.json 2>/dev/null
done

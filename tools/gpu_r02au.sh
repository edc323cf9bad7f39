set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -k "ssnal or multiplier or objective or kkt or path or gap" > gpurun_out/r2au_pytest.log 2>&1; echo rc=$?
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2au_c5_new.json 2>/dev/null
cp abtmp/old_ops.cu paper_2501_15964_b200/csrc/ops.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2au_c5_old.json 2>/dev/null

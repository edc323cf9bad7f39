set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "linf or wide_rows or c4s or project or gap or golden" > gpurun_out/r2ai_pytest.log 2>&1; echo rc=$?
timeout 300 python tools/profile_gamma.py c4inf 0 1 > gpurun_out/r2ai_c4inf_new.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ai_c3_new.json 2>/dev/null
cp abtmp/old_ops.cu paper_2501_15964_b200/csrc/ops.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
timeout 300 python tools/profile_gamma.py c4inf 0 1 > gpurun_out/r2ai_c4inf_old.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ai_c3_old.json 2>/dev/null

set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "gather or ssnal or gap or golden" > gpurun_out/r2ar_pytest.log 2>&1; echo rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ar_c3_new_$i.json 2>/dev/null; done
cp abtmp/old_gather.cu paper_2501_15964_b200/csrc/gather.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ar_c3_old_$i.json 2>/dev/null; done

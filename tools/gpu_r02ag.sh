set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "unchanged or path_parity" > gpurun_out/r2ag_pytest.log 2>&1; echo rc=$?
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2ag_c3_new_$i.json 2>/dev/null
done
cp abtmp/old_solve.cu paper_2501_15964_b200/csrc/solve.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2ag_c3_old_$i.json 2>/dev/null
done

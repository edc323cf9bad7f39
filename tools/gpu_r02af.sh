set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "path or golden or project or warm" > gpurun_out/r2af_pytest.log 2>&1; echo rc=$?
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2af_c3_new_$i.json 2>/dev/null
done
for f in solve.cu ops.cu ops.cuh; do cp abtmp/old_$f paper_2501_15964_b200/csrc/$f; done
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
for i in 1 2; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2af_c3_old_$i.json 2>/dev/null
done

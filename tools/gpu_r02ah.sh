set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "ama or c1 or path or gap" > gpurun_out/r2ah_pytest.log 2>&1; echo rc=$?
for i in 1 2; do timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2ah_c1_$i.json 2>/dev/null; done

set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hessian or linf or l1 or ssnal or path" > gpurun_out/r2n_pytest.log 2>&1; echo pytest rc=$?
timeout 1500 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2n_bench_c4.json 2> gpurun_out/r2n_bench_c4.err; echo c4 rc=$?
timeout 1500 python bench.py --config c4inf --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2n_bench_c4inf.json 2> gpurun_out/r2n_bench_c4inf.err; echo c4inf rc=$?

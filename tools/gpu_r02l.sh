set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x -k "hessian or ssnal or golden or path or tma" > gpurun_out/r2l_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python tools/profile_gamma.py c3 8 12 gpurun_out/r2l_prof.json > gpurun_out/r2l_prof.log 2>&1; echo prof rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2l_bench_c3.json 2> gpurun_out/r2l_bench_c3.err; echo bench rc=$?
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2l_bench_c2.json 2> gpurun_out/r2l_bench_c2.err; echo bench rc=$?

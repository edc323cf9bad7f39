set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hessian or ssnal or path_parity or tma or linf" > gpurun_out/r2i_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python tools/profile_gamma.py c3 0 12 gpurun_out/r2i_prof.json > gpurun_out/r2i_prof.log 2>&1; echo prof rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2i_bench_c3.json 2> gpurun_out/r2i_bench_c3.err; echo bench rc=$?
timeout 1500 python bench.py --config c4inf --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2i_bench_c4inf.json 2> gpurun_out/r2i_bench_c4inf.err; echo c4inf rc=$?

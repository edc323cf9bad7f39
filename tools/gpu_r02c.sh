set -x
make -s -C tests/cpp
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r2c_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2c_bench_c3.json 2> gpurun_out/r2c_bench_c3.err; echo bench rc=$?

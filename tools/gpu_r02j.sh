set -x
make -s -C tests/cpp
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r2j_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2j_bench_c3.json 2> gpurun_out/r2j_bench_c3.err; echo bench rc=$?
timeout 1500 python bench.py --config c4inf --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2j_bench_c4inf.json 2> gpurun_out/r2j_bench_c4inf.err; echo c4inf rc=$?
timeout 300 python tools/profile_path.py c3 20 > gpurun_out/r2j_plain.log 2>&1 && timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2j_launches_c3_full.csv python tools/profile_path.py c3 20 > gpurun_out/r2j_ncu_launch.log 2>&1; echo launches rc=$?

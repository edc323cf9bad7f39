set -x
make -s -C tests/cpp
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/r2h_pytest.log 2>&1; echo pytest rc=$?
timeout 1500 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2h_bench_c4.json 2> gpurun_out/r2h_bench_c4.err; echo c4 rc=$?
timeout 1500 python bench.py --config c4inf --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2h_bench_c4inf.json 2> gpurun_out/r2h_bench_c4inf.err; echo c4inf rc=$?
timeout 1200 python tools/perf_profiles.py c2 60 gpurun_out/r2h_perf_profile_c2 > gpurun_out/r2h_perf_c2.log 2>&1; echo perf rc=$?
timeout 300 python tools/profile_path.py c3 20 > gpurun_out/r2h_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hess_tma -s 150 -c 8 -o gpurun_out/r2h_hess_g10 python tools/profile_path.py c3 20 > gpurun_out/r2h_ncu.log 2>&1; echo ncu rc=$?

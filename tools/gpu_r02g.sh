set -x
timeout 900 python tools/profile_gamma.py c3admm 0 2 gpurun_out/r2g_admm_c3.json 20 > gpurun_out/r2g_admm_c3.log 2>&1; echo admm rc=$?
timeout 1500 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2g_bench_c4.json 2> gpurun_out/r2g_bench_c4.err; echo c4 rc=$?
timeout 1500 python bench.py --config c4inf --steps 1 --warmup 0 --no-e2e --no-cpu --time-limit 15 > gpurun_out/r2g_bench_c4inf.json 2> gpurun_out/r2g_bench_c4inf.err; echo c4inf rc=$?

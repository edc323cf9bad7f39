set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3 rc=$?
python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_c2 rc=$?
python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1 rc=$?
timeout 600 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hess_tma --launch-skip 20 -c 1 -o gpurun_out/ncu_hess_c3_b -f python tools/profile_path.py c3 3 > gpurun_out/ncu_hess_b.log 2>&1; echo ncu_hess_c3 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hess_warp --launch-skip 5 -c 1 -o gpurun_out/ncu_hessw_c5 -f python tools/profile_path.py c5 2 > gpurun_out/ncu_hessw.log 2>&1; echo ncu_hessw_c5 rc=$?

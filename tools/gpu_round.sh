set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3 rc=$?
python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_c2 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
ncu --set full --import-source on -k regex:k_knn_tc -c 1 -o gpurun_out/ncu_knn_c3 python tools/profile_path.py c3 1 > gpurun_out/ncu_knn.log 2>&1; echo knn rc=$?
ncu --set full --import-source on -k regex:k_hess_tma --launch-skip 151 -c 1 -o gpurun_out/ncu_hess_c3 python tools/profile_path.py c3 10 > gpurun_out/ncu_hess.log 2>&1; echo hess rc=$?
ncu --set full --import-source on -k regex:k_mult_t --launch-skip 20 -c 1 -o gpurun_out/ncu_mult_c3 python tools/profile_path.py c3 10 > gpurun_out/ncu_mult.log 2>&1; echo mult rc=$?

# Round-end refresh of the bench lines, the reference arm and the launch list (one GPU).
set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3 rc=$?
python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_c2 rc=$?
python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1 rc=$?
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench_c5 rc=$?
python bench.py --impl reference > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err; echo ref_c3 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?

set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_c3 rc=$?
python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench_c2 rc=$?
python bench.py --impl reference > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err; echo ref_c3 rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?

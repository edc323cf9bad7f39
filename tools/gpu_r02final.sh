set -x
make -s -C tests/cpp
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/fin7_pytest.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/fin7_bench_c3.json 2> gpurun_out/fin7_bench_c3.err; echo c3 rc=$?
timeout 600 python bench.py --config c2 > gpurun_out/fin7_bench_c2.json 2> gpurun_out/fin7_bench_c2.err; echo c2 rc=$?
timeout 600 python bench.py --config c1 > gpurun_out/fin7_bench_c1.json 2> gpurun_out/fin7_bench_c1.err; echo c1 rc=$?
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/fin7_bench_c5.json 2> gpurun_out/fin7_bench_c5.err; echo c5 rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/fin7_ref_c3.json 2> gpurun_out/fin7_ref_c3.err; echo ref rc=$?

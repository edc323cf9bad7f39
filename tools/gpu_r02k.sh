set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_paths.py -m gpu -q -x > gpurun_out/r2k_pytest.log 2>&1; echo pytest rc=$?
timeout 300 python tools/profile_gamma.py c4inf 0 1 - 3 > gpurun_out/r2k_plain.log 2>&1; echo plain rc=$?
for K in k_mult_inf_s k_phi_edge_linf_s k_g_hess k_edge_dot_inf; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o gpurun_out/r2k_$K python tools/profile_gamma.py c4inf 0 1 - 3 > gpurun_out/r2k_ncu_$K.log 2>&1; echo ncu $K rc=$?
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r2k_bench_c3.json 2> gpurun_out/r2k_bench_c3.err; echo bench rc=$?

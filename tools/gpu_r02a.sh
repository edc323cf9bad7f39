set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "^CPU\(s\)|Model name|Thread|Socket"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python tools/profile_gamma.py c3 8 12 gpurun_out/r2a_prof_tma.json > gpurun_out/r2a_prof_tma.log 2>&1; echo rc=$?
CPB_TMA_HESS=0 timeout 600 python tools/profile_gamma.py c3 8 12 gpurun_out/r2a_prof_2pass.json > gpurun_out/r2a_prof_2pass.log 2>&1; echo rc=$?
timeout 300 python tools/profile_path.py c3 20 > gpurun_out/r2a_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hess_tma --launch-skip 150 -c 1 -o gpurun_out/r2a_hess_g10 python tools/profile_path.py c3 20 > gpurun_out/r2a_ncu.log 2>&1; echo ncu rc=$?

set -x
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2m_c2_slot.json 2>/dev/null; echo rc=$?
cp paper_2501_15964_b200/csrc/hess_tma.cu /tmp/hess_slot.cu
cp abtmp/hess_tma_fixedstage.cu paper_2501_15964_b200/csrc/hess_tma.cu
make -s -j16 -C paper_2501_15964_b200/csrc > gpurun_out/r2m_make.log 2>&1; echo make rc=$?
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2m_c2_fixed.json 2>/dev/null; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2m_c3_fixed.json 2>/dev/null; echo rc=$?

set -x
for mb in 3 4 2; do
sed -i "s/__launch_bounds__(256, NP == 1 ? [0-9] : 1) k_hess_warp/__launch_bounds__(256, NP == 1 ? $mb : 1) k_hess_warp/" paper_2501_15964_b200/csrc/gather.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2av_c5_mb$mb.json 2>/dev/null
done

set -x
for nf in 3 4 6; do
sed -i "s/constexpr int nf_max = [0-9];/constexpr int nf_max = $nf;/" paper_2501_15964_b200/csrc/gather.cu
make -s -j16 -C paper_2501_15964_b200/csrc > /dev/null 2>&1; echo make rc=$?
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ao_c3_nf${nf}_$i.json 2>/dev/null; done
done
cp abtmp/old_gather.cu paper_2501_15964_b200/csrc/gather.cu

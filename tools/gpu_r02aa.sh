for ch in 0 4096 2048 1024; do
CPB_TMA_CHUNK=$ch timeout 300 python tools/profile_gamma.py c4inf 0 1 > gpurun_out/r2aa_c4inf_$ch.log 2>&1
done
for ch in 0 2048 1024 512; do
CPB_TMA_CHUNK=$ch timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2aa_c3_$ch.json 2>/dev/null
done

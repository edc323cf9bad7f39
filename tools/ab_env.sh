# A/B environment settings on one library build: bash tools/ab_env.sh <config> <ngamma> "<ENV=..>" ...
set -u
cfg=$1; ng=$2; shift 2
python tools/profile_path.py $cfg 2 > /dev/null 2>&1  # warm the box
for r in 1 2; do
  i=0
  for e in "$@"; do
    i=$((i+1))
    env $e timeout 900 python tools/profile_path.py $cfg $ng stats > gpurun_out/abenv_${cfg}_${i}_$r.txt 2>&1
    echo "$cfg [$e] $r rc=$? $(grep -E 'hess' gpurun_out/abenv_${cfg}_${i}_$r.txt | head -2 | tr -s ' ' | tr '\n' ' ') $(head -1 gpurun_out/abenv_${cfg}_${i}_$r.txt | grep -o 'wall [0-9.]*')"
  done
done

# A/B two builds of the library on the same box: abtmp/libold.so vs abtmp/libnew.so
# usage: bash tools/ab_lib.sh <config> <ngamma> [reps]
set -u
L=paper_2501_15964_b200/libcluspath_b200.so
cfg=$1; ng=$2; reps=${3:-2}
cp abtmp/libnew.so $L; python tools/profile_path.py $cfg 2 > /dev/null 2>&1  # warm the box
for r in $(seq 1 $reps); do
  for v in old new; do
    cp abtmp/lib$v.so $L
    timeout 900 python tools/profile_path.py $cfg $ng stats > gpurun_out/ab_${cfg}_${v}_$r.txt 2>&1
    echo "$cfg $v $r rc=$?"
  done
done
cp abtmp/libnew.so $L

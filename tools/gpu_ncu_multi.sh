# usage: [export BN_...=...;] bash tools/gpu_ncu_multi.sh tag regex1 [regex2 ...]
# plain run, launch list, then one ncu --set full capture per kernel regex
set -x
tag=$1; shift
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$B > gpurun_out/plain_$tag.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$tag.csv $B > /dev/null 2>&1; echo launches rc=$?
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/${tag}_$k $B > gpurun_out/ncu_${tag}_$k.log 2>&1; echo ncu $k rc=$?
done

# C5 (256^2, T = 8192, SWAP): launch list and one ncu --set full capture of the L = 256 cluster decide
set -x
B="python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$B > gpurun_out/plain_c5.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c5.csv $B > /dev/null 2>&1; echo launches_c5 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_decide_big -s 2 -c 1 -o gpurun_out/c5_k_decide_big $B > gpurun_out/ncu_c5_big.log 2>&1; echo ncu c5 big rc=$?

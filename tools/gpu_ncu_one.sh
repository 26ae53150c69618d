# usage: bash tools/gpu_ncu_one.sh <kernel-regex> <outname>   (plain run first, then one ncu --set full)
set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain_$2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$1 -s 2 -c 1 -o gpurun_out/$2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$2.log 2>&1; echo ncu rc=$?

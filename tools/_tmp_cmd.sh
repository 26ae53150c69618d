B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-secondary"
ncu --set full --import-source on --clock-control none -k regex:k_decide_swap -s 6 -c 1 -o gpurun_out/r02_decide_full $B > /dev/null 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_finish_gather -s 6 -c 1 -o gpurun_out/r02_commit_full $B > /dev/null 2>&1; echo rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_decide_big -s 4 -c 1 -o gpurun_out/r02_decide_big_full $B --config C5 > /dev/null 2>&1; echo rc=$?

# round-2 final measurement: every config's bench line, ncu launch lists (C3 SWAP / REDRAW, C5) with
# per-kernel DRAM bytes, and one `ncu --set full` capture of the Gram (C3), each ncu run only after
# the same command exited 0 without ncu
set -x
bash tools/bench_all.sh
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-secondary"
$B > /dev/null 2>&1 && ncu $M -c 200 --log-file gpurun_out/r02f_ncu_C3.csv $B > /dev/null 2>&1; echo c3 rc=$?
$B --mode redraw > /dev/null 2>&1 && ncu $M -c 200 --log-file gpurun_out/r02f_ncu_C3r.csv $B --mode redraw > /dev/null 2>&1; echo c3r rc=$?
$B --config C5 > /dev/null 2>&1 && ncu $M -c 120 --log-file gpurun_out/r02f_ncu_C5.csv $B --config C5 > /dev/null 2>&1; echo c5 rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_gram -s 6 -c 1 -o gpurun_out/r02f_gram_full $B > gpurun_out/r02f_ncu_full.log 2>&1; echo full rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_gram -s 6 -c 1 -o gpurun_out/r02f_gram_full_C5 $B --config C5 > gpurun_out/r02f_ncu_full5.log 2>&1; echo full5 rc=$?

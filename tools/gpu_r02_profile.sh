# round-2 measurement: default bench line, ncu launch lists + per-kernel DRAM bytes (C3 SWAP, C3 REDRAW, C5)
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench rc=$?
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-secondary"
$B > /dev/null 2>&1 && ncu $M -c 200 --log-file gpurun_out/r02_ncu_C3.csv $B > /dev/null 2>&1; echo c3 rc=$?
$B --mode redraw > /dev/null 2>&1 && ncu $M -c 200 --log-file gpurun_out/r02_ncu_C3r.csv $B --mode redraw > /dev/null 2>&1; echo c3r rc=$?
$B --config C5 > /dev/null 2>&1 && ncu $M -c 120 --log-file gpurun_out/r02_ncu_C5.csv $B --config C5 > /dev/null 2>&1; echo c5 rc=$?

# round 2: full GPU suite with the full-size goldens, then the default bench line
set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -30 > gpurun_out/r02a_pytest.log; echo pytest rc=$?
tail -30 gpurun_out/r02a_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/r02a_bench.json; tail -3 gpurun_out/r02a_bench.err
nproc; lscpu | grep "Model name"

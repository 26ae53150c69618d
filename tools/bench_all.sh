# every BASELINE config on one GPU (+ the reference arm on C3); JSON lines -> gpurun_out/bench_all.jsonl
set -x
out=gpurun_out/bench_all.jsonl; : > $out
python bench.py --steps 20 --warmup 5 >> $out 2> gpurun_out/bench_C3.err; echo C3 rc=$?
python bench.py --config C1 --steps 200 --warmup 5 --cpu-classes 64 >> $out 2> gpurun_out/bench_C1.err; echo C1 rc=$?
python bench.py --config C2 --steps 50 --warmup 5 --cpu-classes 16 >> $out 2> gpurun_out/bench_C2.err; echo C2 rc=$?
python bench.py --config C4 --steps 10 --warmup 3 --cpu-classes 8 >> $out 2> gpurun_out/bench_C4.err; echo C4 rc=$?
python bench.py --config C5 --steps 5 --warmup 3 --cpu-classes 1 --e2e-steps 2 >> $out 2> gpurun_out/bench_C5.err; echo C5 rc=$?
python bench.py --impl reference --steps 5 --warmup 3 >> $out 2> gpurun_out/bench_ref.err; echo ref rc=$?
nproc; lscpu | grep "Model name"

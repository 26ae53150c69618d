# Round-1 refresh: every config's bench line (+ alternate modes), the reference arm, the C3 launch list
# and ncu --set full captures of the C3 kernels.  Outputs under gpurun_out/.
set -x
out=gpurun_out/bench_all.jsonl; : > $out
python bench.py --steps 20 --warmup 5 >> $out 2> gpurun_out/bench_C3.err; echo C3 rc=$?
python bench.py --config C3 --mode redraw --steps 20 --warmup 5 --cpu-classes 12 >> $out 2> gpurun_out/bench_C3r.err; echo C3r rc=$?
python bench.py --config C3 --mode paper --steps 20 --warmup 5 --cpu-classes 16 >> $out 2> gpurun_out/bench_C3p.err; echo C3p rc=$?
python bench.py --config C1 --steps 200 --warmup 5 --cpu-classes 64 >> $out 2> gpurun_out/bench_C1.err; echo C1 rc=$?
python bench.py --config C1 --mode swap --steps 200 --warmup 5 --cpu-classes 64 >> $out 2> gpurun_out/bench_C1s.err; echo C1s rc=$?
python bench.py --config C2 --steps 50 --warmup 5 --cpu-classes 16 >> $out 2> gpurun_out/bench_C2.err; echo C2 rc=$?
python bench.py --config C2 --mode paper --steps 50 --warmup 5 --cpu-classes 16 >> $out 2> gpurun_out/bench_C2p.err; echo C2p rc=$?
python bench.py --config C4 --steps 10 --warmup 3 --cpu-classes 8 >> $out 2> gpurun_out/bench_C4.err; echo C4 rc=$?
python bench.py --config C4 --mode redraw --steps 10 --warmup 3 --cpu-classes 8 >> $out 2> gpurun_out/bench_C4r.err; echo C4r rc=$?
python bench.py --config C5 --steps 5 --warmup 3 --cpu-classes 1 --e2e-steps 2 >> $out 2> gpurun_out/bench_C5.err; echo C5 rc=$?
python bench.py --config C5 --mode redraw --steps 5 --warmup 3 --cpu-classes 1 --e2e-steps 2 >> $out 2> gpurun_out/bench_C5r.err; echo C5r rc=$?
python bench.py --config C3 --mode redraw --K 4 --steps 5 --warmup 3 --cpu-classes 2 --e2e-steps 2 >> $out 2> gpurun_out/bench_C3k4.err; echo C3k4 rc=$?
python bench.py --impl reference --steps 5 --warmup 3 >> $out 2> gpurun_out/bench_ref.err; echo ref rc=$?
nproc; lscpu | grep "Model name"
bash tools/gpu_ncu_multi.sh r01z k_gram_tc4 k_decide_swap k_lut k_finish_gather
bash tools/gpu_ncu_c5.sh
ls gpurun_out

# every BASELINE config on one GPU (+ the reference arm on C3); JSON lines -> gpurun_out/r02_bench_all.jsonl
out=gpurun_out/r02_bench_all.jsonl; : > $out
python bench.py --steps 20 --warmup 5 >> $out 2> gpurun_out/r02_all_C3.err; echo C3 rc=$?
python bench.py --steps 20 --warmup 5 --mode redraw --no-secondary >> $out 2> gpurun_out/r02_all_C3r.err; echo C3r rc=$?
python bench.py --steps 20 --warmup 5 --mode paper --no-secondary >> $out 2> gpurun_out/r02_all_C3p.err; echo C3p rc=$?
python bench.py --steps 5 --warmup 3 --mode redraw --K 4 --no-secondary --cpu-classes 2 --e2e-steps 4 >> $out 2> gpurun_out/r02_all_C3k.err; echo C3k rc=$?
python bench.py --config C1 --steps 200 --warmup 5 --cpu-classes 64 --no-secondary >> $out 2> gpurun_out/r02_all_C1.err; echo C1 rc=$?
python bench.py --config C1 --mode swap --steps 200 --warmup 5 --cpu-classes 64 --no-secondary >> $out 2> gpurun_out/r02_all_C1s.err; echo C1s rc=$?
python bench.py --config C2 --steps 50 --warmup 5 --cpu-classes 16 --no-secondary >> $out 2> gpurun_out/r02_all_C2.err; echo C2 rc=$?
python bench.py --config C2 --mode paper --steps 50 --warmup 5 --cpu-classes 16 --no-secondary >> $out 2> gpurun_out/r02_all_C2p.err; echo C2p rc=$?
python bench.py --config C4 --steps 10 --warmup 3 --cpu-classes 8 --no-secondary >> $out 2> gpurun_out/r02_all_C4.err; echo C4 rc=$?
python bench.py --config C4 --mode redraw --steps 10 --warmup 3 --cpu-classes 8 --no-secondary >> $out 2> gpurun_out/r02_all_C4r.err; echo C4r rc=$?
python bench.py --config C5 --steps 5 --warmup 3 --cpu-classes 1 --e2e-steps 4 --no-secondary >> $out 2> gpurun_out/r02_all_C5.err; echo C5 rc=$?
python bench.py --config C5 --mode redraw --steps 5 --warmup 3 --cpu-classes 1 --e2e-steps 4 --no-secondary >> $out 2> gpurun_out/r02_all_C5r.err; echo C5r rc=$?
python bench.py --impl reference --steps 5 --warmup 3 >> $out 2> gpurun_out/r02_all_ref.err; echo ref rc=$?

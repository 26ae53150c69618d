# parity on all decide/gram variants + bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
BN_DECIDE=flags timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or c3_shape or radii" 2>&1 | tail -1
BN_GRAM=imma2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c3_shape or shard" 2>&1 | tail -1; BN_DECIDE=per_class BN_GRAM=simt timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or c2 or c3_shape or shard" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print('value', d['value'], 'ms/step', d['ms_per_step']); print('kernels', d['kernels_ms_per_step']); print('roof', d['roofline']['kernel'], d['roofline']['frac']); print('e2e', d['e2e']['value'])
"
tail -3 gpurun_out/bench_q.err

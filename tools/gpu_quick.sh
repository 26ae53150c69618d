# quick GPU check: parity tests then a short bench (used during development)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print('value', d['value'], 'ms/step', d['ms_per_step']); print('kernels', d['kernels_ms_per_step']); print('roof', d['roofline']); print('e2e', d['e2e']['value'])
"
tail -3 gpurun_out/bench_q.err

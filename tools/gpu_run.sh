# usage: bash tools/gpu_run.sh TAG [pytest-args...]: GPU suite (+ default bench line) -> gpurun_out/TAG_*
tag=$1; shift
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${tag}_pytest.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/${tag}_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/${tag}_bench.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value']); print(d['kernels_ms_per_step'])" 2>&1 | tail -3
tail -3 gpurun_out/${tag}_bench.err

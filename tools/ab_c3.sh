# usage: bash tools/ab_c3.sh "ENV1" "ENV2" ...   C3 bench (20 steps) once per env setting, twice each
for e in "$@"; do for i in 1 2; do
  env $e python bench.py --steps 20 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value']/1e6,2), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()})"
done; done

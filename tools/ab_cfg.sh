# usage: bash tools/ab_cfg.sh CONFIG STEPS "ENV1" "ENV2" ...   one bench line per env setting
cfg=$1; steps=$2; shift 2
for e in "$@"; do
  env $e python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline --e2e-steps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$e', round(d['value']/1e6,3), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()})"
done

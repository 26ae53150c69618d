# usage: bash tools/ab_env.sh "ENV1=a ENV2=b" "ENV1=c" ... [-- bench args]: one bench line per env set
args="--steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 4"
sets=()
while [ $# -gt 0 ]; do
  if [ "$1" = "--" ]; then shift; args="$args $*"; break; fi
  sets+=("$1"); shift
done
for e in "${sets[@]}"; do
  env $e python bench.py $args > /tmp/ab.json 2> /tmp/ab.err || { echo "$e: FAILED"; tail -2 /tmp/ab.err; continue; }
  python - "$e" <<'PY'
import json, sys
d = json.load(open("/tmp/ab.json"))
k = {a: round(b * 1e3, 1) for a, b in d["kernels_ms_per_step"].items()}
print(f"{sys.argv[1]:>28}: {d['value']/1e6:7.2f} M evals/s  {d['ms_per_step']*1e3:6.1f} us/pass  e2e {d['e2e']['value']/1e6:6.2f}  {k}")
PY
done

# parity tests + A/B runs; usage: RUNS='name|ENV=1 ENV2=2|--bench-args;...' bash scripts/gpu_ab.sh TAG
TAG=${1:-ab}
[ -z "$NO_PYTEST" ] && timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
run() {  # name, env string, bench args
  local name=$1 envs=$2 args=$3
  env $envs timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $args > gpurun_out/${TAG}_${name}.json 2>gpurun_out/${TAG}_${name}.err
  python - "$name" gpurun_out/${TAG}_${name}.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(f"{sys.argv[1]:>12}", 'value', round(d['value']), 'ms/step', round(d['ms_per_step'], 4), 'frac', round(d['roofline']['frac'], 3), 'kernel_ms', {k: round(v, 4) for k, v in d['roofline']['kernel_ms'].items()})
except Exception as e:
    print(sys.argv[1], 'FAILED', e)
PY
  tail -2 gpurun_out/${TAG}_${name}.err
}
IFS=';' read -ra R <<< "${RUNS:-base||}"
for spec in "${R[@]}"; do
  IFS='|' read -r n e a <<< "$spec"
  run "$n" "$e" "$a"
done

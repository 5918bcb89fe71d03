# e2e A/B: bench with e2e (no cpu baseline) for the default build and variants; usage: VARIANTS="a b" bash scripts/gpu_e2e_ab.sh TAG [bench args]
TAG=$1; shift
L=paper_1904_01201_b200/_lib/variants
for v in base $VARIANTS; do
  if [ "$v" = base ]; then E=""; else E="NAVSIM_B200_LIB=$L/libnavsim_$v.so"; fi
  env $E timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-eval "$@" > gpurun_out/${TAG}_$v.json 2>gpurun_out/${TAG}_$v.err
  python - "$v" gpurun_out/${TAG}_$v.json <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    print(f"{sys.argv[1]:>10} value {d['value']/1e6:.3f}M  us/step {d['ms_per_step']*1e3:.1f}  e2e {d['e2e']['value']/1e6:.3f}M ({1024/d['e2e']['value']*1e6 if d['e2e'] else 0:.1f} us/step)")
except Exception as e:
    print(sys.argv[1], 'FAILED', e)
PY
done

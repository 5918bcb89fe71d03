# parity tests + bench (quick iteration).  usage: bash scripts/gpu_quick.sh TAG [pytest-args]
TAG=${1:-q}
shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > gpurun_out/${TAG}_pytest.txt 2>&1
tail -25 gpurun_out/${TAG}_pytest.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('value', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'step_frac', round(d['roofline']['step_frac'],3), 'kernel_ms', {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, 'e2e', d['e2e'] and round(d['e2e']['value']), 'clocks', d['clocks'])
"

# parity tests + bench (quick iteration)
TAG=${1:-q}
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('value', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['roofline']['kernel'][:14], 'kernel_ms', {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, 'e2e', d['e2e'] and round(d['e2e']['value']), 'clocks', d['clocks'])
"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --cast-mode 1 > gpurun_out/${1:-q}_bench_fused.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/${1:-q}_bench_fused.json'))
print('BINNED-CAST value', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'kernel_ms', {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})
"
if [ -f paper_1904_01201_b200/_lib/libnavsim_b200_rw4.so ]; then
NAVSIM_B200_LIB=$PWD/paper_1904_01201_b200/_lib/libnavsim_b200_rw4.so timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/${1:-q}_bench_rw4.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/${1:-q}_bench_rw4.json'))
print('RW4 value', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'kernel_ms', {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})
"
fi

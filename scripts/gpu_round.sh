# full round check: parity tests, smoke, default bench (+cpu baseline), binned-cast A/B, launch list
TAG=${1:-r1b}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/${TAG}_pytest_gpu.txt
tail -8 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 8 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --cast-mode 1 > gpurun_out/${TAG}_bench_binned.json 2>/dev/null; cat gpurun_out/${TAG}_bench_binned.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err; cat gpurun_out/${TAG}_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/${TAG}_launches.csv

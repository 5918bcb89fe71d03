# full round check: parity tests, smoke, default bench (+cpu baseline), reference arm, launch list, ncu full
TAG=${1:-r1}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/${TAG}_pytest_gpu.txt
tail -4 gpurun_out/${TAG}_pytest_gpu.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 8 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -3 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err; cat gpurun_out/${TAG}_bench_ref.json
for C in C1 C2 C4 C5; do timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$C.json 2> gpurun_out/${TAG}_bench_$C.err; tail -1 gpurun_out/${TAG}_bench_$C.err; head -c 600 gpurun_out/${TAG}_bench_$C.json; echo; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-graph --no-e2e --no-cpu-baseline > /dev/null 2>&1
NCU_COUNT=3 bash scripts/gpu_ncu_one.sh ${TAG} 'k_column_cast|k_agent_step|k_fill_ws'

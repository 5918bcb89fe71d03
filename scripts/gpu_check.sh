set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/r1_pytest_gpu.txt
cat gpurun_out/r1_pytest_gpu.txt | tail -25
timeout 300 python __graft_entry__.py 2>&1 | tail -5
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-seconds 8 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err; tail -3 gpurun_out/r1_bench.err; cat gpurun_out/r1_bench.json

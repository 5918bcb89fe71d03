TAG=${1:-pa}
B="python bench.py --steps 3 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"k_agent_step" -s 3 -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log

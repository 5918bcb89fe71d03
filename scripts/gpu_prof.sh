# ncu launch list + full capture of the cast and fill kernels (one GPU)
TAG=${1:-r1}
B="python bench.py --steps 4 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_column_cast|k_fill_tma|k_agent_step" -s 6 -c 3 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
ls -la gpurun_out

TAG=${1:-r3}
KR=${2:-k_column_cast}
B="python bench.py --steps 4 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s 2 -c 1 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log

# one ncu --set full capture of the kernels matching $2 (bench args in $3)
TAG=${1:-p}; KR=${2:-k_fill}; ARGS=${3:-}
B="python bench.py --steps 3 --warmup 3 --no-graph --no-e2e --no-cpu-baseline $ARGS"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s 3 -c ${NCU_COUNT:-1} -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log

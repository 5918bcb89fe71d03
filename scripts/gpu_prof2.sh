TAG=${1:-r2}
python scripts/write_bw.py > gpurun_out/${TAG}_writebw.json; cat gpurun_out/${TAG}_writebw.json
B="python bench.py --steps 4 --warmup 3 --no-graph --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_column_cast|k_fill_tma" -s 4 -c 2 -o gpurun_out/${TAG}_prof $B > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log

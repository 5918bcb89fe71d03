TAG=${1:-x3}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for C in C3 C2; do timeout 600 python scripts/step_breakdown.py $C > gpurun_out/${TAG}_breakdown_$C.json 2>&1; cat gpurun_out/${TAG}_breakdown_$C.json; echo; done
NO_PYTEST=1 RUNS="c3||;c2||--config C2;c1||--config C1;c4||--config C4;c5||--config C5" bash scripts/gpu_ab.sh $TAG
python -c "import bench; print(bench.cpu_baseline('C3', seconds=8.0, threads=1)['value'], bench.cpu_baseline('C3', seconds=8.0)['value'])"

TAG=${1:-x2}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 900 python scripts/bench_simulator.py > gpurun_out/${TAG}_simulator.json 2> gpurun_out/${TAG}_simulator.err; tail -3 gpurun_out/${TAG}_simulator.err; cat gpurun_out/${TAG}_simulator.json; echo
timeout 600 python scripts/step_breakdown.py C3 > gpurun_out/${TAG}_breakdown_c3.json 2>&1; cat gpurun_out/${TAG}_breakdown_c3.json; echo
timeout 600 python scripts/step_breakdown.py C2 > gpurun_out/${TAG}_breakdown_c2.json 2>&1; cat gpurun_out/${TAG}_breakdown_c2.json; echo
timeout 900 python scripts/eval_pointgoal.py C5 512 64 200 > gpurun_out/${TAG}_pointgoal_c5.json 2> gpurun_out/${TAG}_pointgoal_c5.err; tail -3 gpurun_out/${TAG}_pointgoal_c5.err; cat gpurun_out/${TAG}_pointgoal_c5.json

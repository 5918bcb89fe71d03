# round-2 measurement rows: C5 PointGoal eval, single-env Simulator facade vs the reference, reference anchor
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python scripts/eval_pointgoal.py C5 512 64 200 > gpurun_out/${TAG}_pointgoal_c5.json 2> gpurun_out/${TAG}_pointgoal_c5.err; tail -2 gpurun_out/${TAG}_pointgoal_c5.err; head -c 1500 gpurun_out/${TAG}_pointgoal_c5.json; echo
timeout 900 python scripts/bench_simulator.py > gpurun_out/${TAG}_simulator.json 2> gpurun_out/${TAG}_simulator.err; tail -2 gpurun_out/${TAG}_simulator.err; cat gpurun_out/${TAG}_simulator.json; echo
[ -z "$NO_ANCHOR" ] && timeout 1500 python scripts/ref_anchor.py > gpurun_out/${TAG}_ref_anchor.json 2> gpurun_out/${TAG}_ref_anchor.err; tail -2 gpurun_out/${TAG}_ref_anchor.err; head -c 3000 gpurun_out/${TAG}_ref_anchor.json

# the A/B runs of gpu_ab.sh without the parity tests
NO_PYTEST=1 RUNS="$RUNS" bash scripts/gpu_ab.sh "$1"

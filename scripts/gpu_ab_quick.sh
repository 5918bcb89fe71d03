sed '/pytest/d' scripts/gpu_ab.sh > /tmp/ab.sh; RUNS="$RUNS" bash /tmp/ab.sh "$1"

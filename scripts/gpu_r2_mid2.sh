#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
O=gpurun_out/r2_mid2.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O 2>&1
echo "tests rc=$?" >> $O
J=gpurun_out/r2_mid2.jsonl
: > $J
timeout 600 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat20 --k 4 5 6 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $J 2>&1
timeout 900 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $J 2>&1
echo done >> $J
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat20_k7_mid.csv \
  python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>&1

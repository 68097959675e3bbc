#!/bin/bash
# iteration 2: full GPU suite + pivot split / per-lane S-tier timings + exact peel
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs KC_GQ_DEBUG=1
O=gpurun_out/r2_iter2.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O 2>&1
echo "tests rc=$?" >> $O
J=gpurun_out/r2_iter2.jsonl
: > $J
timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy --reps 2 >> $J 2>&1
for sp in 0 16 64; do
  echo "{\"pivot_split\": $sp}" >> $J
  KC_PIVOT_SPLIT=$sp timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy --reps 1 >> $J 2>&1
done
timeout 900 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $J 2>&1
timeout 300 python scripts/exact_order_check.py rmat18 rmat22 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat18 --k 4 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $J 2>&1
echo done >> $J
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat20_k7.csv \
  python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/r2_launches_rmat20_k7.log 2>&1

#!/bin/bash
# dynamic pair loops (orient) + spill rounds (pivot): GPU suite, headline,
# RMAT-22 k=7 slice, RMAT-18 k=10 / k=7 pivot, budget sweep
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_dyn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_dyn_tests.log
export KC_TIMING=1
O=gpurun_out/r2b_dyn.log
: > $O
timeout 300 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 64 --ranks 0 >> $O 2>&1
echo "rc=$?" >> $O
timeout 900 python scripts/explore.py --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 600 python scripts/explore.py --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
for B in 131072 32768; do
  echo "{\"budget\": $B}" >> $O
  KC_SPILL_BUDGET=$B timeout 300 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
  echo "rc=$?" >> $O
done

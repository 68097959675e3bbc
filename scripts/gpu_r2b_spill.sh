#!/bin/bash
# pivot bounded walks + spill rounds: GPU suite, then RMAT-14/16 k=10 (exact
# visits), a budget sweep, and the heaviest RMAT-18 k=10 shard
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_spill_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_spill_tests.log
export KC_TIMING=1
O=gpurun_out/r2b_spill.log
: > $O
timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy --reps 2 >> $O 2>&1
echo "rc=$?" >> $O
for B in 65536 8192 524288; do
  echo "{\"budget\": $B}" >> $O
  KC_SPILL_BUDGET=$B timeout 300 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
  echo "rc=$?" >> $O
done
timeout 400 python scripts/shard_probe.py --workload rmat18 --k 10 --algo pivot --scheme edge --world 128 --ranks 0 >> $O 2>&1
echo "rc=$?" >> $O

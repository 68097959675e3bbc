#!/bin/bash
# pivot hand-over policy sweep (RMAT-14/16 k=10, reference heap order)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs KC_GQ_DEBUG=1
J=gpurun_out/r2_pivot_tune.jsonl
: > $J
for cfg in "12 256 4" "12 256 0" "12 64 0" "12 16 0" "8 16 0" "6 16 0" "12 4 0" "24 16 0"; do
  set -- $cfg
  echo "{\"push_min\": $1, \"cooldown\": $2, \"room\": $3}" >> $J
  KC_GQ_PUSHMIN=$1 KC_GQ_COOLDOWN=$2 KC_GQ_ROOM=$3 timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy --reps 2 >> $J 2>&1
  KC_GQ_PUSHMIN=$1 KC_GQ_COOLDOWN=$2 KC_GQ_ROOM=$3 timeout 600 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $J 2>&1
done
echo done >> $J

#!/bin/bash
# north-star target on one GPU: RMAT-20 / RMAT-22 k=7 (orientation, reference heap order)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
J=gpurun_out/r2_rmat22_k7.jsonl
: > $J
timeout 900 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $J 2>&1
timeout 3300 python scripts/explore.py --workload rmat22 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $J 2>&1
echo "rc=$?" >> $J

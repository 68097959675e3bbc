#!/bin/bash
# full RMAT-22 ef16 k=7 (orientation, vertex, reference heap order) on one GPU
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs KC_TIMING=1
O=gpurun_out/r2b_rmat22_k7.log
: > $O
timeout 2400 python scripts/explore.py --workload rmat22 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O

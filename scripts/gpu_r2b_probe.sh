#!/bin/bash
# where the time goes at HEAD: per-launch device times (KC_TIMING) for
# RMAT-20 k=7 orient, RMAT-16 k=10 pivot; shard slices of RMAT-22 k=7 and RMAT-18 k=10
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs KC_TIMING=1
O=gpurun_out/r2b_probe.log
: > $O
timeout 400 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 600 python scripts/shard_probe.py --workload rmat18 --k 10 --algo pivot --scheme edge --world 32 --ranks 0 16 31 >> $O 2>&1
echo "rc=$?" >> $O
timeout 900 python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 16 --ranks 0 8 15 >> $O 2>&1
echo "rc=$?" >> $O

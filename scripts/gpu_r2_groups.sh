#!/bin/bash
# sub-warp group sizes: correctness + A/B timing of the orientation warp tier
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
O=gpurun_out/r2_groups.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "group or small_suite or medium or closed or split or shard" > $O 2>&1
echo "tests rc=$?" >> $O
J=gpurun_out/r2_groups.jsonl
: > $J
timeout 900 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --group 32 16 8 4 2 1 --reps 2 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat16 --k 8 --algo orient --scheme vertex --criterion degeneracy --group 32 8 2 1 --reps 2 >> $J 2>&1
echo done >> $J

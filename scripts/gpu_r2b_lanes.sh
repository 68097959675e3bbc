#!/bin/bash
# per-lane pivot walk: lanes filled by the actual child bound, shared loads,
# no kernel-parameter address taken; GPU suite + spill test + timings
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_lanes_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_lanes_tests.log
export KC_TIMING=1
O=gpurun_out/r2b_lanes.log
: > $O
timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy --reps 2 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $O 2>&1
echo "rc=$?" >> $O
timeout 1200 python scripts/explore.py --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O

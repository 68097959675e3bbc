#!/bin/bash
# RMAT-22 k=7 root ranges: orientation vs pivot (timed), then the test;
# RMAT-18 k=10 vertex scheme; ncu of a pivot spill-round launch after the lane fixes
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
O=gpurun_out/r2b_x.log
: > $O
for R in "0 1500" "600000 640000" "2000000 2395364"; do
  for A in orient pivot; do
    timeout 300 python scripts/shard_probe.py --workload rmat22 --k 7 --algo $A --scheme vertex --range $R >> $O 2>&1
    echo "rc=$?" >> $O
  done
done
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k rmat22_root_ranges --durations=5 > gpurun_out/r2b_x_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_x_tests.log
KC_TIMING=1 timeout 900 python scripts/explore.py --workload rmat18 --k 10 --algo pivot --scheme vertex --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 1 \
  --launch-skip 5 -o gpurun_out/r2b_pivot_round3_rmat16_v2 -f \
  python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 > gpurun_out/r2b_ncu_pivot2.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_ncu_pivot2.log

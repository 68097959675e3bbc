#!/bin/bash
# ncu --set full: pivot spill-round warp launch (RMAT-16 k=10, round 3) and the
# headline warp-tier launch (RMAT-18 k=7 triples)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
python scripts/explore.py --workload rmat16 --k 4 --reps 1 > /dev/null 2>&1
python scripts/explore.py --workload rmat18 --k 4 --reps 1 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 1 \
  --launch-skip 5 -o gpurun_out/r2b_pivot_round3_rmat16 -f \
  python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 > gpurun_out/r2b_ncu_pivot.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_ncu_pivot.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 1 \
  -o gpurun_out/r2b_orient_triples_rmat18 -f \
  python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/r2b_ncu_orient.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_ncu_orient.log

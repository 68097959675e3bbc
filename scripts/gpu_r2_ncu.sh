#!/bin/bash
# ncu --set full: orientation warp tier at RMAT-18 k=7 (triples + items launches) and the
# pivot warp tier at RMAT-14 k=10 (heap order)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
python -c "
from paper_2104_13209_b200 import synth; import numpy as np, os
os.makedirs('/tmp/kc_graphs', exist_ok=True)
for w in ('rmat14', 'rmat18'): np.save(f'/tmp/kc_graphs/{w}.npy', synth.workload(w))"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 2 -o gpurun_out/r2_orient_rmat18_k7 -f \
  python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/r2_ncu_orient.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu_orient.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 1 -o gpurun_out/r2_pivot_rmat14_k10 -f \
  python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 > gpurun_out/r2_ncu_pivot.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu_pivot.log

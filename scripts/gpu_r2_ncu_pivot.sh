#!/bin/bash
# ncu --set full of the pivot warp-tier kernel (RMAT-14 k=10, heap order) + pivot policy sweep
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
python -c "from paper_2104_13209_b200 import synth; import numpy as np, os; os.makedirs('/tmp/kc_graphs', exist_ok=True); np.save('/tmp/kc_graphs/rmat14.npy', synth.workload('rmat14'))"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 1 -o gpurun_out/r2_pivot_rmat14_k10 -f \
  python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 > gpurun_out/r2_ncu_pivot.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu_pivot.log
bash scripts/gpu_r2_pivot_tune.sh

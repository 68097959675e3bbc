#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
python -c "from paper_2104_13209_b200 import synth; import numpy as np, os; os.makedirs('/tmp/kc_graphs', exist_ok=True); np.save('/tmp/kc_graphs/rmat18.npy', synth.workload('rmat18'))"
timeout 900 ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats --section SchedulerStats --section SourceCounters --section ComputeWorkloadAnalysis \
   --clock-control none --import-source on -k regex:'k_count<' -c 1 -o gpurun_out/prof_cta_k7_r18 \
   python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>> gpurun_out/ncu.err
echo done

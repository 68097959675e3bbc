#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pivot7.csv \
    python scripts/explore.py --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1 > gpurun_out/pivot7.log 2>&1
echo done

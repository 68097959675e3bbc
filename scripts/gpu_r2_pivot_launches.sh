#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs KC_GQ_DEBUG=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat16_k10_pivot.csv \
  python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 > gpurun_out/r2_pivot_launches.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat14_k10_pivot_vertex.csv \
  python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme vertex --criterion degeneracy --reps 1 >> gpurun_out/r2_pivot_launches.log 2>&1

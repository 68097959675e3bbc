#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
export PYTHONPATH=$PWD
timeout 1850 python scripts/explore.py --workload rmat22 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/rmat22_k7.log 2>&1
echo "rc=$?" >> gpurun_out/rmat22_k7.log
echo done

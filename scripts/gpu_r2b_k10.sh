#!/bin/bash
# adaptive spill budget, larger item buffers: spill test, headline check,
# full RMAT-18 k=10 (pivot, edge) with per-round progress
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests/test_gpu_spill.py -q -x > gpurun_out/r2b_k10_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_k10_tests.log
export KC_TIMING=1
O=gpurun_out/r2b_k10.log
: > $O
timeout 300 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $O 2>&1
echo "rc=$?" >> $O
timeout 1500 python scripts/explore.py --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O

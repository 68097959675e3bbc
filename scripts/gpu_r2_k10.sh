#!/bin/bash
# k=10 pivot under the reference's heap order: RMAT-16, RMAT-18
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GQ_DEBUG=1
O=gpurun_out/r2_k10.jsonl
: > $O
timeout 300 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy --reps 1 >> $O 2>&1
timeout 1500 python scripts/explore.py --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo done >> $O

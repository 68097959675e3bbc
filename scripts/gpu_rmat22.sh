#!/bin/bash
# BASELINE config 5 workload on one GPU: RMAT scale-22 ef16, k=7, degeneracy
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
E=gpurun_out/explore_rmat22.jsonl
: > $E
timeout 2100 python scripts/explore.py --workload rmat22 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $E 2>> gpurun_out/explore22.err
echo "{\"rc\": $?}" >> $E
echo done

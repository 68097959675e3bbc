#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=60 run --workload rmat18 --k 4 --algo orient --scheme vertex --criterion degeneracy degree --reps 3
T=300 run --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:k_count -c 2 -o gpurun_out/prof_orient7_r18 \
   python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>> gpurun_out/ncu.err
T=900 run --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
echo done

#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=60 run --workload rmat12 --k 7 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
export KC_GQ=1 KC_GQ_DEBUG=1
T=60 run --workload rmat12 --k 7 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=90 run --workload rmat14 --k 7 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=120 run --workload rmat16 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1
timeout 200 python -m pytest tests -m gpu -x -q -k "pivot or medium or small or shards" > gpurun_out/pytest_gq.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gq.log
echo done

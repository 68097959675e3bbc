#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
export KC_GQ_DEBUG=1
T=150 run --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=100 run --workload rmat16 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=100 run --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=60 run --workload rmat18 --k 4 --algo pivot --scheme edge --criterion degeneracy --reps 1
echo done

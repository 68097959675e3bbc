#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=100 run --workload rmat18 --k 5 6 7 --algo orient --scheme vertex --criterion degeneracy --reps 2
T=100 run --workload rmat16 --k 7 --algo orient --scheme vertex edge --criterion degeneracy --reps 2
echo done

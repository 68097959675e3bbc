#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=200 run --workload rmat14 --k 7 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=300 run --workload rmat16 --k 7 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=200 run --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=600 run --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
timeout 600 ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats --section SchedulerStats --section SourceCounters --section ComputeWorkloadAnalysis \
   --clock-control none --import-source on -k k_count -c 1 -o gpurun_out/prof_cta_k7_r18 \
   python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/ncu_cta.log 2>&1
echo done

#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_r1e.json 2>> gpurun_out/bench_r1e.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=100 run --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=150 run --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=900 run --workload rmat18 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
echo done

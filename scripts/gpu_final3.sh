#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
KC_GQ=0 timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_nogq.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_nogq.log
timeout 900 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count -c 2 -o gpurun_out/prof_final_r16b \
   python scripts/explore.py --workload rmat16 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/ncu_f.log 2>&1
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=100 run --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1
T=150 run --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 1
echo done

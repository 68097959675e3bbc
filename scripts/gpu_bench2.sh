#!/bin/bash
# bench line (k=7 headline + per_k 4/7/10), reference arm, launch list, ncu of the top kernel
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 1500 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r1.json 2>> gpurun_out/bench_r1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
echo done

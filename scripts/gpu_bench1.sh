#!/bin/bash
# first bench + ncu evidence of the working path (k=4, RMAT-18, degeneracy)
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_k4.json 2> gpurun_out/bench_k4.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 --cpu-sample-s 6 > gpurun_out/bench_ref_k4.json 2>> gpurun_out/bench_k4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k4.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>> gpurun_out/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -s 1 -c 1 -o gpurun_out/prof_k4 \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>> gpurun_out/ncu.err
echo done

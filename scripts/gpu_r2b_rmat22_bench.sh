#!/bin/bash
# north-star config through bench.py: RMAT-22 ef16 k=7, one timed step (a
# step is ~16 min; no warm-up: the library has no JIT), e2e, roofline, CPU baseline
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 3300 python bench.py --workload rmat22 --k 7 --steps 1 --warmup 0 --per-k 7 --no-configs \
  > gpurun_out/r2b_bench_rmat22.json 2> gpurun_out/r2b_bench_rmat22.err
echo "rc=$?" >> gpurun_out/r2b_bench_rmat22.err

#!/bin/bash
# round-2 evidence: default bench line (RMAT-18 k=7 headline, per_k 4/7/10,
# side configs, CPU baseline, e2e), the reference arm, then the north-star
# config RMAT-22 ef16 k=7 through bench.py (1 warm-up + 1 step: ~16 min each)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2b_final_smi.txt 2>&1
timeout 2400 python bench.py > gpurun_out/r2b_final_bench.json 2> gpurun_out/r2b_final_bench.err
echo "rc=$?" >> gpurun_out/r2b_final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2b_final_bench_ref.json 2> gpurun_out/r2b_final_bench_ref.err
echo "rc=$?" >> gpurun_out/r2b_final_bench_ref.err
timeout 4200 python bench.py --workload rmat22 --k 7 --steps 1 --warmup 1 --per-k 4,7 --no-configs \
  > gpurun_out/r2b_final_bench_rmat22.json 2> gpurun_out/r2b_final_bench_rmat22.err
echo "rc=$?" >> gpurun_out/r2b_final_bench_rmat22.err

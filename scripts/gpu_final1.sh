#!/bin/bash
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_r1b.json 2>> gpurun_out/bench_r1b.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k k_count_warp -c 1 -o gpurun_out/prof_warp_k7_r18 \
   python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/ncu_w.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_count -c 1 -o gpurun_out/prof_cta_k7_r18 \
   python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/ncu_c.log 2>&1
echo done

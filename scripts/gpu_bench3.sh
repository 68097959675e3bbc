#!/bin/bash
# round-1 evidence: bench line (k=7 headline + per_k 4/7), reference arm,
# launch list of the bench command, ncu --set full of the count kernels
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_r1.json 2>> gpurun_out/bench_r1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count -c 3 -o gpurun_out/prof_orient7_r16 \
   python scripts/explore.py --workload rmat16 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>> gpurun_out/ncu.err
echo done

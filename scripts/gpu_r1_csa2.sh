#!/bin/bash
# CSA everywhere in the orient pair loops: parity suite, smoke, bench, reference arm,
# headline launch list, one full capture of the warp-tier kernel (RMAT-16 k=7).
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
export PYTHONPATH=$PWD
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_k7.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_warp -c 1 -o gpurun_out/prof_warp_r16 \
   python scripts/explore.py --workload rmat16 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 > gpurun_out/ncu_f.log 2>&1
echo done

#!/bin/bash
# Round-1 final evidence on the committed build: parity suite, smoke, bench, reference arm, launch list.
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
export PYTHONPATH=$PWD
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2>> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final_k7.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-configs --per-k 7 > /dev/null 2>> gpurun_out/ncu.err
echo done

#!/bin/bash
# re-entry check of HEAD: GPU suite, smoke, default bench line
mkdir -p gpurun_out
export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2b_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_smoke.log
timeout 1200 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "rc=$?" >> gpurun_out/r2b_bench.err

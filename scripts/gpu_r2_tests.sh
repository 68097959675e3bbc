#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpu_tests.log

#!/bin/bash
# one gpurun call: GPU tests + a first sweep of the configs (each bounded)
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
E=gpurun_out/explore.jsonl
: > $E
run() { timeout ${T:-120} python scripts/explore.py "$@" >> $E 2>> gpurun_out/explore.err; echo "{\"rc\": $?, \"args\": \"$*\"}" >> $E; }
T=60 run --workload er2000 --k 4 --oracle-workers 8
T=120 run --workload rmat18 --k 4 --algo orient pivot --scheme vertex edge --criterion degree degeneracy
T=200 run --workload rmat18 --k 7 --algo orient --scheme vertex edge --criterion degeneracy
T=200 run --workload rmat18 --k 7 --algo pivot --scheme vertex edge --criterion degeneracy
T=200 run --workload rmat18 --k 10 --algo pivot --scheme vertex edge --criterion degeneracy
T=120 run --workload planted --k 10 --algo pivot --scheme vertex edge --criterion degeneracy --all-k
T=200 run --workload rmat20 --k 4 7 --algo orient --scheme vertex edge --criterion degeneracy

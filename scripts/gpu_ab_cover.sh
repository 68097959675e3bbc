#!/bin/bash
# A/B: pivot cover popcount with carry-save accumulation (new) vs per-word POPC (old).
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
export PYTHONPATH=$PWD
L=paper_2104_13209_b200
cp $L/libkc_new.so $L/libkc.so
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_ab.log
for v in new old new; do
  cp $L/libkc_$v.so $L/libkc.so
  echo "== $v" >> gpurun_out/ab_cover.log
  timeout 300 python scripts/explore.py --workload rmat16 --k 7 --algo pivot --scheme edge --criterion degeneracy --reps 2 >> gpurun_out/ab_cover.log 2>&1
  timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> gpurun_out/ab_cover.log 2>&1
done
cp $L/libkc_new.so $L/libkc.so
echo done

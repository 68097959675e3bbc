#!/bin/bash
# parallel-bit-extract compression in the CTA pair level: GPU suite, timings, ncu
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_cmp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_cmp_tests.log
export KC_TIMING=1
O=gpurun_out/r2b_cmp.log
: > $O
timeout 300 python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 64 --ranks 0 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
unset KC_TIMING
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -c 1 \
  --launch-skip 3 -o gpurun_out/r2b_cta_orient_rmat22_v2 -f \
  python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 4096 --ranks 0 > gpurun_out/r2b_ncu_cta2.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_ncu_cta2.log

#!/bin/bash
# build/walk split + overflow size histogram (KC_TIMING), and an ncu capture
# of the CTA-tier orientation kernel on a 1/4096 slice of RMAT-22 k=7
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs KC_TIMING=1
O=gpurun_out/r2b_probe2.log
: > $O
timeout 300 python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 64 --ranks 0 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 200 python scripts/explore.py --workload rmat16 --k 10 --algo pivot --scheme edge --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O
timeout 400 python scripts/shard_probe.py --workload rmat18 --k 10 --algo pivot --scheme edge --world 128 --ranks 0 >> $O 2>&1
echo "rc=$?" >> $O
unset KC_TIMING
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count -c 1 \
  --launch-skip 3 -o gpurun_out/r2b_cta_orient_rmat22 -f \
  python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 4096 --ranks 0 > gpurun_out/r2b_ncu_cta.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_ncu_cta.log

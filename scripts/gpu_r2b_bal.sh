#!/bin/bash
# balanced pair loops (pairs spread evenly over lanes): GPU suite, headline, RMAT-22 slice, RMAT-20 k=7
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_bal_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_bal_tests.log
export KC_TIMING=1
O=gpurun_out/r2b_bal.log
: > $O
timeout 300 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 64 --ranks 0 >> $O 2>&1
echo "rc=$?" >> $O
timeout 300 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $O 2>&1
echo "rc=$?" >> $O

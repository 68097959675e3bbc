#!/bin/bash
# pivot frames relative to the walk's first frame: GPU suite, then RMAT-22
# k=7 range [0, 1500) pivot vs orientation (7,846,284,762,132)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_fix_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_fix_tests.log
O=gpurun_out/r2b_fix.log
: > $O
timeout 400 python scripts/shard_probe.py --workload rmat22 --k 7 --algo pivot --scheme vertex --range 0 1500 >> $O 2>&1
echo "rc=$?" >> $O

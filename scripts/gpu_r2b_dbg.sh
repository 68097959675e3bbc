#!/bin/bash
# pivot/vertex k=7 on RMAT-22 root range [0, 1500): histogram sanity, with
# and without spill rounds, and with the subtree queue off
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
O=gpurun_out/r2b_dbg.log
: > $O
for E in "KC_SPILL=1" "KC_SPILL=0" "KC_SPILL=0 KC_GQ=0"; do
  echo "{\"env\": \"$E\"}" >> $O
  env $E timeout 400 python scripts/shard_probe.py --workload rmat22 --k 7 --algo pivot --scheme vertex --range 0 1500 >> $O 2>&1
  echo "rc=$?" >> $O
done

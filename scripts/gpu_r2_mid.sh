#!/bin/bash
# CTA-tier pair level compressed to <= 128-member 16-byte rows: parity + timings
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
O=gpurun_out/r2_mid.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O 2>&1
echo "tests rc=$?" >> $O
J=gpurun_out/r2_mid.jsonl
: > $J
timeout 600 python scripts/explore.py --workload rmat18 --k 4 7 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat20 --k 4 5 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat22 --k 4 --algo orient --scheme vertex --criterion degeneracy --reps 2 >> $J 2>&1
timeout 900 python scripts/explore.py --workload rmat20 --k 7 --algo orient --scheme vertex --criterion degeneracy --reps 1 >> $J 2>&1
echo done >> $J

#!/bin/bash
# round-2 exploration: exact heap-order peel cost and pivot trees under it
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
export PYTHONPATH=$PWD
O=gpurun_out/r2_explore1.jsonl
: > $O
timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge vertex --criterion degeneracy_exact degeneracy --reps 1 >> $O 2>&1
timeout 300 python scripts/explore.py --workload rmat18 --k 4 --algo orient --scheme vertex --criterion degeneracy_exact degeneracy --reps 2 >> $O 2>&1
timeout 300 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy_exact degeneracy --reps 1 >> $O 2>&1
timeout 600 python scripts/explore.py --workload rmat18 --k 7 --algo pivot --scheme edge --criterion degeneracy_exact --reps 1 >> $O 2>&1
timeout 300 python scripts/explore.py --workload rmat22 --k 4 --algo orient --scheme vertex --criterion degeneracy_exact degeneracy --reps 1 >> $O 2>&1
echo done >> $O

#!/bin/bash
# iteration: parity subset + A/B timings + launch lists (k=4 RMAT-18, k=5 RMAT-20)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
O=gpurun_out/r2_iter.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > $O 2>&1
echo "tests rc=$?" >> $O
J=gpurun_out/r2_iter.jsonl
: > $J
timeout 600 python scripts/explore.py --workload rmat18 --k 7 --algo orient --scheme vertex --criterion degeneracy degeneracy_bulk --group 32 1 --reps 2 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat18 --k 4 5 6 --algo orient --scheme vertex --criterion degeneracy --group 32 --reps 3 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat16 --k 8 --algo orient --scheme vertex --criterion degeneracy --group 32 1 --reps 2 >> $J 2>&1
timeout 600 python scripts/explore.py --workload rmat20 --k 5 --algo orient --scheme vertex edge --criterion degeneracy --group 32 --reps 2 >> $J 2>&1
echo done >> $J
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat20_k5.csv \
  python scripts/explore.py --workload rmat20 --k 5 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat18_k4.csv \
  python scripts/explore.py --workload rmat18 --k 4 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat22_k4.csv \
  python scripts/explore.py --workload rmat22 --k 4 --algo orient --scheme vertex --criterion degeneracy --reps 1 > /dev/null 2>&1

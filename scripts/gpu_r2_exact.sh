#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
O=gpurun_out/r2_exact.log
python -m pytest tests/test_gpu_parity.py -x -q -k "exact or degeneracy or medium" > $O 2>&1
timeout 900 python scripts/exact_order_check.py rmat14 rmat16 rmat18 rmat20 rmat22 >> $O 2>&1
timeout 300 python scripts/explore.py --workload rmat14 --k 10 --algo pivot --scheme edge --criterion degeneracy_exact --reps 2 >> $O 2>&1
echo done >> $O

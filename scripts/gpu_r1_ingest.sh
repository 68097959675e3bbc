#!/bin/bash
# K0 ingest: GPU tests (new + full suite), smoke, bench line with the ingest side measurement.
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
timeout 300 python -m pytest tests/test_ingest.py -m gpu -x -q > gpurun_out/pytest_ingest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ingest.log
timeout 400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
# launch list of the ingest kernels alone
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ingest_launches.csv python -c "
import numpy as np, paper_2104_13209_b200 as kc
from paper_2104_13209_b200 import synth
raw = synth.rmat_raw(20, 16, seed=1)
kc.normalize_edges(raw)
" > gpurun_out/ingest_ncu.log 2>&1
echo done

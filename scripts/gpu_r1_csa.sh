#!/bin/bash
# CSA pair loops: GPU parity suite, smoke, bench; ingest launch list + full capture of k_orient_pack.
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
export PYTHONPATH=$PWD
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat > /tmp/ingest_one.py <<'PY'
import numpy as np, paper_2104_13209_b200 as kc
from paper_2104_13209_b200 import synth
raw = synth.rmat_raw(20, 16, seed=1)
g = kc.from_raw_edges(raw)
print(g.n, g.m, g.n_self_loops, g.n_duplicates)
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ingest_launches.csv python /tmp/ingest_one.py > gpurun_out/ingest_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_orient_pack -c 1 -o gpurun_out/ingest_pack python /tmp/ingest_one.py > gpurun_out/ingest_full.log 2>&1
echo done

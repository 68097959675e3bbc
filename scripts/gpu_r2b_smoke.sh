#!/bin/bash
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke_final.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_smoke_final.log

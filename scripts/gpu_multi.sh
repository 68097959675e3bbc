#!/bin/bash
# N>1 code path of bench.py on a 1-GPU box: 2 ranks share cuda:0 over gloo
mkdir -p gpurun_out
export KC_GRAPH_CACHE=/tmp/kc_graphs
KC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 \
    > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
echo "rc=$?" >> gpurun_out/bench_2rank.err
KC_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --cpu-sample-s 3 \
    > gpurun_out/bench_2rank_ref.json 2>> gpurun_out/bench_2rank.err
echo done

#!/bin/bash
# round-2 evidence: A/B of the compressed pair-level cap on a RMAT-22 k=7
# slice (counts must agree), the default bench line (RMAT-18 k=7 headline,
# per_k 4/7/10, side configs, CPU baseline, e2e), the reference arm, then the
# north-star config RMAT-22 ef16 k=7 through bench.py (1 warm-up + 1 step)
mkdir -p gpurun_out
export PYTHONPATH=$PWD KC_GRAPH_CACHE=/tmp/kc_graphs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2b_final_smi.txt 2>&1
O=gpurun_out/r2b_final_ab.log
: > $O
for M in 256 128; do
  KC_MID_MAX=$M timeout 400 python scripts/shard_probe.py --workload rmat22 --k 7 --algo orient --scheme vertex --world 64 --ranks 0 > gpurun_out/ab_$M.json 2>&1
  echo "{\"mid_max\": $M}" >> $O; cat gpurun_out/ab_$M.json >> $O
done
MID=$(python - <<'PY'
import json
def last(p):
    for l in reversed(open(p).read().splitlines()):
        if l.startswith('{"rank"'): return json.loads(l)
try:
    a, b = last('gpurun_out/ab_256.json'), last('gpurun_out/ab_128.json')
    print(128 if (a["count"] == b["count"] and b["kernel_ms"] < 0.97 * a["kernel_ms"]) else 256)
except Exception:
    print(256)
PY
)
echo "{\"chosen_mid_max\": $MID}" >> $O
export KC_MID_MAX=$MID
timeout 2400 python bench.py > gpurun_out/r2b_final_bench.json 2> gpurun_out/r2b_final_bench.err
echo "rc=$?" >> gpurun_out/r2b_final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2b_final_bench_ref.json 2> gpurun_out/r2b_final_bench_ref.err
echo "rc=$?" >> gpurun_out/r2b_final_bench_ref.err
timeout 4200 python bench.py --workload rmat22 --k 7 --steps 1 --warmup 1 --per-k 4,7 --no-configs \
  > gpurun_out/r2b_final_bench_rmat22.json 2> gpurun_out/r2b_final_bench_rmat22.err
echo "rc=$?" >> gpurun_out/r2b_final_bench_rmat22.err

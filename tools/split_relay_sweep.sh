#!/usr/bin/env bash
# Exploration: HS_PROG_SPLIT_RELAY variants vs the current best at N ranks (variant_probe).
N=${1:-2}; OUT=${2:-gpurun_out/split_n$N.jsonl}
P=29640
for w in cfg2e cfg2a cfg2b cfg2d cfg3b cfg3a; do
  timeout 300 torchrun --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P++)) tools/variant_probe.py \
    --workload $w --flags 16789504,12288,1073745920,1090523136,1073741824,536883200 --steps 100 2>&1 | grep '^{' >> $OUT
done
for share in 24 40; do
  HS_SPLIT_RELAY_64THS=$share timeout 300 torchrun --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P++)) \
    tools/variant_probe.py --workload cfg2e --flags 1073745920,1090523136 --steps 100 2>&1 | grep '^{' | \
    sed "s/^{/{\"share64\": $share, /" >> $OUT
done

#!/usr/bin/env bash
# Exploration: split relay combined with interleaved items (and static dealing) vs the
# current best variants, at N ranks (variant_probe, per-rank phase times).
N=${1:-2}; OUT=${2:-gpurun_out/split_interleave_n$N.jsonl}
P=29970
for w in cfg2e cfg2a cfg2b cfg2d cfg3b cfg3a; do
  timeout 300 torchrun --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((P++)) tools/variant_probe.py \
    --workload $w --flags 16789504,12288,1073745920,1610616832,1627394048,536883200 --steps 100 2>&1 | grep '^{' >> $OUT
done

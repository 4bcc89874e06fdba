#!/usr/bin/env bash
# Exploration: untuned program variants for the switch workloads at N ranks
# (bench.py --config W --flags F --no-tune), to pick StrategyCycle's default.
N=${1:-2}; OUT=${2:-gpurun_out/switch_defaults_n$N.jsonl}
P=29850
for w in cfg4 cfg5_S1S2 cfg5_S2S3 cfg5_S3S4 cfg5_S4S1; do
  for f in 1024 33555584 570425472 570426496; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((P++)) bench.py --gpus $N --config $w --steps 10 --warmup 3 --no-switch --no-cpu \
      --no-tune --e2e-steps 1 --flags $f 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
print(json.dumps({'workload': '$w', 'n': $N, 'flags': $f, 'ms': d['ms_per_step'], 'verified': d['verified']}))" >> $OUT
  done
done

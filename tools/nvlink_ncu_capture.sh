#!/usr/bin/env bash
# NVLink / DRAM counters of a multi-GPU program, one profiled rank at a time
# (see tools/nvlink_ncu_capture.py).  Usage:
#   tools/nvlink_ncu_capture.sh WORKLOAD FLAGS WORLD PROFILED_RANK OUT_PREFIX [LAUNCHES_PER_RUN]
set -u
WL=${1:-cfg2e}; FLAGS=${2:-0}; WORLD=${3:-2}; PR=${4:-0}; OUT=${5:-gpurun_out/nvl}
NPH=${6:-2}   # data-kernel launches per run (plan phases launched)
WARM=5        # tools/nvlink_ncu_capture.py --warmup default
METRICS=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
export WORLD_SIZE=$WORLD MASTER_ADDR=127.0.0.1 MASTER_PORT=$((29500 + RANDOM % 400))
pids=()
for ((r = 0; r < WORLD; r++)); do
  if [[ $r == "$PR" ]]; then
    RANK=$r timeout 240 ncu -k regex:box_phase --launch-skip $((WARM * NPH)) --launch-count $NPH --clock-control none \
      --metrics "$METRICS" --csv --log-file "${OUT}_r${r}.csv" \
      python tools/nvlink_ncu_capture.py --workload "$WL" --flags "$FLAGS" --profiled-rank "$PR" \
      > "${OUT}_r${r}.log" 2>&1 &
  else
    RANK=$r timeout 240 python tools/nvlink_ncu_capture.py --workload "$WL" --flags "$FLAGS" \
      --profiled-rank "$PR" > "${OUT}_r${r}.log" 2>&1 &
  fi
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait "$p" || rc=1; done
exit $rc

#!/usr/bin/env bash
# diagnostic: which ncu filter profiles a kernel of a 2-rank run (rank 1 profiled)
set -u
export WORLD_SIZE=2 MASTER_ADDR=127.0.0.1
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
run() {  # name, ncu args...
  local name=$1; shift
  export MASTER_PORT=$((29500 + RANDOM % 400))
  RANK=0 timeout 100 python tools/nvlink_ncu_capture.py --flags 16789504 --profiled-rank 1 > gpurun_out/diag_${name}_r0.log 2>&1 &
  local p0=$!
  RANK=1 timeout 100 ncu "$@" --metrics $M --csv --log-file gpurun_out/diag_${name}_r1.csv \
    python tools/nvlink_ncu_capture.py --flags 16789504 --profiled-rank 1 > gpurun_out/diag_${name}_r1.log 2>&1
  echo "$name rc=$?"
  wait $p0; echo "$name r0 rc=$?"
}
run first3 -c 3
run regex -k regex:box_phase -c 4
run tail -k regex:tail -c 2

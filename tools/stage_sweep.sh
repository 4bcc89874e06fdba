#!/usr/bin/env bash
# Exploration: TMA pipeline geometry (stages x stage KB) of the executor kernels.
# Builds one library per geometry under paper_2504_20490_b200/lib/variants/ (run here,
# before gpurun), then on the GPU times cfg2e / cfg3b / cfg4 / cfg5 S1->S2 at N=1 with each
# (HS_LIB_VARIANT selects the library; tools/variant_probe.py, flags 0).
#   tools/stage_sweep.sh build        # CPU container
#   tools/stage_sweep.sh run OUT      # GPU box
set -u
GEOMS="4x48 4x56 6x32 3x64 5x40"
if [[ ${1:-} == build ]]; then
  for g in $GEOMS; do
    st=${g%x*}; kb=${g#*x}
    make -s -C paper_2504_20490_b200/csrc -j16 EXTRA_DEFS="-DHS_TMA_STAGES=$st -DHS_STAGE_KB=$kb" \
      OUTDIR=../lib/variants/$g BUILD=../lib/variants/$g/obj ../lib/variants/$g/libhshard_b200.so
  done
  exit 0
fi
OUT=${2:-gpurun_out/stage_sweep.jsonl}
for g in $GEOMS; do
  for w in cfg2e cfg3b cfg2b; do
    HS_LIB_VARIANT=$g timeout 300 python tools/variant_probe.py --workload $w --flags 0 --steps 200 2>&1 | \
      grep '^{' | sed "s/^{/{\"geom\": \"$g\", /" >> $OUT
  done
done

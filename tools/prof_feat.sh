#!/bin/bash
# Full ncu captures (source level) of feature-stage kernels in the 16-pair 1024^2 pipeline.
mkdir -p gpurun_out
for K in "$@"; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o gpurun_out/full_feat_$K \
      python tools/stage_timing.py --pairs 16 --iters 2 > gpurun_out/full_feat_$K.log 2>&1
  echo "$K rc=$?"
  ncu -i gpurun_out/full_feat_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_feat_$K.csv 2>/dev/null
done

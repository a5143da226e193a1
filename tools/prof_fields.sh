#!/bin/bash
# Full ncu captures (source-level) of the filter-bank kernels, one launch each.
# usage: tools/prof_fields.sh TAG [kernel regex...]
TAG=${1:?tag}; shift
mkdir -p gpurun_out
make -C paper_2303_00319_b200/csrc -j16 > /dev/null 2>&1
for K in "${@:-k_rows_pc_tma k_cols}"; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o gpurun_out/full_${TAG}_${K} \
      python tools/fields_timing.py --size 1024 --pairs 16 --iters 2 > gpurun_out/full_${TAG}_${K}.log 2>&1
  echo "$K rc=$?"
  ncu -i gpurun_out/full_${TAG}_${K}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_${TAG}_${K}.csv 2>/dev/null
  ncu -i gpurun_out/full_${TAG}_${K}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_${K}.csv 2>/dev/null
done

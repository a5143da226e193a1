#!/bin/bash
# Full ncu capture of k_match_gemm (tensor pipe metrics) in the bench's batch and at C4.
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_match_gemm -s 1 -c 1 -o gpurun_out/full_gemm_c2 \
    python tools/stage_timing.py --pairs 16 --iters 2 > gpurun_out/full_gemm_c2.log 2>&1
echo "c2 rc=$?"
ncu --set full --clock-control none -k regex:k_match_gemm -c 1 -o gpurun_out/full_gemm_c4 \
    python tools/stage_timing.py --pairs 1 --size 4096 --max-kp 20000 --iters 1 > gpurun_out/full_gemm_c4.log 2>&1
echo "c4 rc=$?"
for t in c2 c4; do
  ncu -i gpurun_out/full_gemm_$t.ncu-rep --page raw --csv > gpurun_out/raw_gemm_$t.csv 2>/dev/null
done

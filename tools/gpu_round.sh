#!/bin/bash
# One round-end measurement call on the GPU box: GPU tests, bench line, launch
# list and --set full captures of the top kernels.  usage: tools/gpu_round.sh TAG
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 bash tools/launches.sh $TAG > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 bash tools/prof_feat.sh k_desc_main k_match_gemm > /dev/null 2>&1; echo "feat captures rc=$?"

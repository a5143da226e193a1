#!/bin/bash
# Round-end measurement on the GPU box (one gpurun call):
#   1. bench.py (the JSON line the driver also produces)
#   2. the ncu launch list of the same command (time + DRAM bytes per launch)
#   3. one --set full capture of the top kernel
# usage: tools/round_profile.sh TAG [TOP_KERNEL_REGEX]
set -u
TAG=${1:?tag}; TOP=${2:-k_rows_pc}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || { tail -5 gpurun_out/bench_$TAG.err; exit 1; }
cat gpurun_out/bench_$TAG.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 \
    --csv --log-file gpurun_out/bench_launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_ncu_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:$TOP -s 2 -c 1 -o gpurun_out/full_$TAG \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full_ncu_$TAG.log 2>&1
echo "full capture rc=$?"

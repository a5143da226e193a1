#!/bin/bash
# Per-kernel launch list of one pipeline iteration (run on the GPU box).
# usage: tools/launches.sh TAG [pairs]
TAG=${1:-x}; PAIRS=${2:-16}
# our kernels per pipeline iteration (BatchPipeline.KERNELS_PER_STEP): skip one iteration, capture one
PER=${PER:-$(python -c "from paper_2303_00319_b200.batch import BatchPipeline as B; print(B.KERNELS_PER_STEP)")}
mkdir -p gpurun_out
python tools/stage_timing.py --pairs $PAIRS --iters 2 --size ${SIZE:-1024} --max-kp ${MAXKP:-5000} > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum \
    --clock-control none -k regex:^k_ -s $PER -c $PER --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/stage_timing.py --pairs $PAIRS --iters 2 --size ${SIZE:-1024} --max-kp ${MAXKP:-5000} > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/plain_$TAG.log

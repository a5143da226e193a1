#!/bin/bash
# Per-kernel ncu times of one filter-bank pass for library variants.
# usage: tools/kernel_times.sh "NAME:FLAGS" ...
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  out=/tmp/var_$name
  make -C paper_2303_00319_b200/csrc -j16 OUT_DIR=$out EXTRA_NVFLAGS="$flags" > /tmp/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
  RIFT2_B200_LIB=$out/librift2_b200.so ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none -k regex:^k_ -s 27 -c 9 --csv --log-file gpurun_out/kt_$name.csv \
     python tools/fields_timing.py --size 1024 --pairs 16 --iters 2 > /dev/null 2>&1
  echo "== $name"; python tools/show_launches.py gpurun_out/kt_$name.csv 1
done

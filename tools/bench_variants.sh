#!/bin/bash
# Build library variants (EXTRA_NVFLAGS) and run the bench's pipelined step with each.
# usage: tools/bench_variants.sh "NAME1:-DFOO=1" ...
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  out=/tmp/var_$name
  make -C paper_2303_00319_b200/csrc -j16 OUT_DIR=$out EXTRA_NVFLAGS="$flags" > /tmp/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
  RIFT2_B200_LIB=$out/librift2_b200.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-other-configs > gpurun_out/bv_$name.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/bv_$name.json'))
print('$name', 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'fb_ms', round(d['roofline']['launch_ms'],3), 'frac', round(d['roofline']['frac'],3))"
done

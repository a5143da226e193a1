#!/bin/bash
# Build library variants (EXTRA_NVFLAGS) and time the filter bank with each.
# usage: tools/variants.sh "NAME1:-DFOO=1" "NAME2:-DFOO=2" ...
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  out=/tmp/var_$name
  make -C paper_2303_00319_b200/csrc -j16 OUT_DIR=$out EXTRA_NVFLAGS="$flags" > /tmp/build_$name.log 2>&1 || { echo "$name build failed"; tail -3 /tmp/build_$name.log; continue; }
  for sz in "1024 16" ${EXTRA_SIZES}; do
    set -- $sz
    RIFT2_B200_LIB=$out/librift2_b200.so python tools/fields_timing.py --size $1 --pairs $2 | sed "s/^/$name /"
  done
done

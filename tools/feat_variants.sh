#!/bin/bash
# Build library variants and print the two-stream timeline (tools/timeline.py) with each.
# usage: tools/feat_variants.sh "NAME1:-DFOO=1" ...
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}; out=/tmp/var_$name
  make -C paper_2303_00319_b200/csrc -j16 OUT_DIR=$out EXTRA_NVFLAGS="$flags" > /tmp/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
  RIFT2_B200_LIB=$out/librift2_b200.so python tools/timeline.py 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['features_alone']
print('$name', 'detect', round(a['detect_end'],3), 'describe', round(a['describe_end']-a['detect_end'],3), 'match', round(a['match_end']-a['describe_end'],3), 'fields', d['fields_alone']['fields_end'], 'both', d['both']['match_end'], d['both']['fields_end'])"
done

#!/bin/bash
# k_match_gemm alone (tools/gemm_only.py) for library variants, e.g.
#   tools/gemm_exp.sh "cur:" "noepi:-DR2_EXP_NOEPI" "loads:-DR2_EXP_NOEPI -DR2_EXP_NOMMA"
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}; out=/tmp/var_$name
  make -C paper_2303_00319_b200/csrc -j16 OUT_DIR=$out EXTRA_NVFLAGS="$flags" > /tmp/build_$name.log 2>&1 || { echo "$name build failed"; grep -m3 -i error /tmp/build_$name.log; continue; }
  echo "$name $(RIFT2_B200_LIB=$out/librift2_b200.so python tools/gemm_only.py 2>&1 | tail -1)"
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in bx128 bx64 bx32; do
  echo "=== $v" >> $O/opbench30.log
  HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg 4 --reps 6 --only apply,vcycle >> $O/opbench30.log 2>&1
done

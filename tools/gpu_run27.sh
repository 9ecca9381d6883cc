#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in s1 s3 s4; do
  for c in 4 2; do
    echo "=== $v cfg$c" >> $O/opbench27.log
    HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench27.log 2>&1
  done
done
tail -3 $O/pytest_gpu26.log > /dev/null

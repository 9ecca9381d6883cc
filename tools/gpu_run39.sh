#!/bin/bash
# operator CTAs of 128 x 2 / 128 x 4 nodes (adjacent lines share gathered rows in L1) vs 128 x 1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for c in 4 2; do
  for v in default tx256 tx512; do
    echo "=== cfg$c $v" >> $O/opbench39.log
    if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
    HJB_LIB=$L timeout 400 python tools/opbench.py --cfg $c --reps 6 --only apply,vcycle >> $O/opbench39.log 2>&1
  done
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test tools/tma_test.cu > $O/tma22.log 2>&1
for a in "6 32 8 0 0" "6 16 8 0 0" "6 32 8 0 1" "6 64 8 1 0" "6 32 8 1 1" "6 8 8 0 1" "6 36 7 0 1"; do timeout 60 ./tools/tma_test $a >> $O/tma22.log 2>&1; echo "exit $?" >> $O/tma22.log; done
for v in ilp1 ilp2 ilp2b; do
  echo "=== $v" >> $O/opbench22.log
  HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg 4 --reps 6 --only apply,vcycle >> $O/opbench22.log 2>&1
done

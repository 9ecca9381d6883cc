#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test tools/tma_test.cu > $O/tma23.log 2>&1
for a in "6 36 7 0 1 8 3" "6 36 7 0 1 9 3" "6 36 7 0 1 297 3" "6 36 7 0 1 296 60" "6 36 7 0 1 8 60" "6 36 7 0 1 8 61" "6 36 7 0 1 2 121"; do timeout 60 ./tools/tma_test $a >> $O/tma23.log 2>&1; echo "exit $?" >> $O/tma23.log; done

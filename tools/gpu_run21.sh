#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test tools/tma_test.cu > $O/tma21.log 2>&1
for m in 3 0 1 2 4 5; do timeout 60 ./tools/tma_test $m >> $O/tma21.log 2>&1; echo "exit $?" >> $O/tma21.log; done

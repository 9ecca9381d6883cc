#!/bin/bash
# ncu --set full of the cfg4 control search (the top kernel with the W-cycle)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
CMD="python tools/opbench.py --cfg 4 --reps 10 --only search"
timeout 600 $CMD > $O/plain52.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_search" -s 0 -c 6 -o $O/prof52_cfg4 $CMD > $O/ncu52.log 2>&1
echo "ncu exit $?" >> $O/ncu52.log

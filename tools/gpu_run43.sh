#!/bin/bash
# ncu --set full of the fine-level smoothing sweeps of one cfg4 V-cycle (from the last OP_DIAG setup launches on)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
CMD="python tools/opbench.py --cfg 4 --reps 2 --only vcycle"
timeout 600 $CMD > $O/plain43.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator|k_jacobi0_diag" -s 28 -c 30 -o $O/prof43_cfg4 $CMD > $O/ncu43.log 2>&1
echo "ncu exit $?" >> $O/ncu43.log

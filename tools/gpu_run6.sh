#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply or policy or cfg0 or inexact" > $O/pytest_gpu6.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu6.log
for v in opA opB opC srB; do
  echo "=== $v" >> $O/opbench6_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 4 --reps 10 >> $O/opbench6_cfg4.log 2>&1
done

#!/bin/bash
# L2 prefetch of the gather band's leading edge: kernel timing at cfg4 (+ parity with the default build)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in nopf pf pf_opB; do
  echo "=== $v" >> $O/opbench10_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 4 --reps 6 >> $O/opbench10_cfg4.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu10.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu10.log

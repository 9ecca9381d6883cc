#!/bin/bash
# block-shape / L1-carveout variants of the 2D-grid kernels: kernel timing at cfg4 + parity on one
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in base bx32 bx64 l1max bx32l1; do
  echo "=== $v" >> $O/opbench9_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 4 --reps 6 >> $O/opbench9_cfg4.log 2>&1
done
HJB_LIB=build_variants/bx32.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q -k "apply or policy or bitwise" > $O/pytest_gpu9.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu9.log

#!/bin/bash
# lean fast-path geometry (floor split, warp-uniform dispatch, smem control tables): variants at cfg4
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in fA fB fC fD; do
  echo "=== $v" >> $O/opbench12_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 4 --reps 6 >> $O/opbench12_cfg4.log 2>&1
done
for v in fA fD; do
  echo "=== $v cfg3" >> $O/opbench12_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 3 --reps 10 >> $O/opbench12_cfg4.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu12.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu12.log

#!/bin/bash
# search variants (unroll2 / minB), full-size parity, bench cfg4 default, ncu launch list of a cfg2 step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in sr1 sr2 sr2b; do
  echo "=== $v" >> $O/opbench7_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 4 --reps 4 --only search >> $O/opbench7_cfg4.log 2>&1
  echo "=== $v cfg3" >> $O/opbench7_cfg4.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 3 --reps 10 --only search >> $O/opbench7_cfg4.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_gpu7.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu7.log
timeout 900 python bench.py --steps 1 --warmup 1 --json-out $O/bench7_cfg4.json > $O/bench7_cfg4.log 2>&1; echo "exit $?" >> $O/bench7_cfg4.log

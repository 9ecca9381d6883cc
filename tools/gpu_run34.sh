#!/bin/bash
# window search with control split: bit identity + timing variants (threads x split)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build34.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu34a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu34a.log
for c in 3 2 1; do
  echo "=== cfg$c w512s2 (default)" >> $O/opbench34.log
  timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench34.log 2>&1
  echo "=== cfg$c direct" >> $O/opbench34.log
  HJB_WIN=0 timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench34.log 2>&1
  for v in w256s1 w512s1 w768s3 w1024s4; do
    echo "=== cfg$c $v" >> $O/opbench34.log
    HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench34.log 2>&1
  done
done
for v in w768s3 w1024s4; do
  HJB_LIB=build_variants/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu34_$v.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu34_$v.log
done

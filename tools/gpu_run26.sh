#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for v in d4 d5 d6 d8; do
  echo "=== $v" >> $O/opbench26.log
  HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg 4 --reps 6 --only apply,vcycle >> $O/opbench26.log 2>&1
done
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build26.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_gpu26.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu26.log

#!/bin/bash
# cfg4 control search (now the top kernel with the W-cycle): register / block-shape variants; all GPU tests
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build47.log 2>&1
for v in default sdeep3 sdeep5 sbx16 sbx64; do
  echo "=== cfg4 $v" >> $O/opbench47.log
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  HJB_LIB=$L timeout 300 python tools/opbench.py --cfg 4 --reps 30 --only search >> $O/opbench47.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu47.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu47.log

#!/bin/bash
# windowed control search: correctness + timing
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build14.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window" > $O/pytest_gpu14a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu14a.log
for c in 4 2 1; do
  echo "=== cfg$c win" >> $O/opbench14.log
  timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench14.log 2>&1
  echo "=== cfg$c direct" >> $O/opbench14.log
  HJB_NO_WINSEARCH=1 timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench14.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest_gpu14.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu14.log

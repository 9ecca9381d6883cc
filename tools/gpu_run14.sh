#!/bin/bash
# windowed control search + deep-rectangle operator kernels: correctness + timing
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build14.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "window" > $O/pytest_gpu14a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu14a.log
for c in 4 2 1 3; do
  echo "=== cfg$c new" >> $O/opbench14.log
  timeout 300 python tools/opbench.py --cfg $c --reps 6 >> $O/opbench14.log 2>&1
  echo "=== cfg$c no-win/no-deep" >> $O/opbench14.log
  HJB_NO_WINSEARCH=1 timeout 300 python tools/opbench.py --cfg $c --reps 6 >> $O/opbench14.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu14.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu14.log

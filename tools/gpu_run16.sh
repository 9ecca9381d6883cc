#!/bin/bash
# TMA-windowed control search: correctness (bit identity) + timing
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build16.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu16a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu16a.log
for c in 4 2 1; do
  echo "=== cfg$c tma" >> $O/opbench16.log
  timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench16.log 2>&1
  echo "=== cfg$c no-tma" >> $O/opbench16.log
  HJB_NO_TMA=1 timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench16.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu16.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu16.log

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build24.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu24a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu24a.log
for c in 4 2; do
  echo "=== cfg$c tma" >> $O/opbench24.log
  timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench24.log 2>&1
  echo "=== cfg$c no-tma" >> $O/opbench24.log
  HJB_NO_TMA=1 timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench24.log 2>&1
done
timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > $O/bench24.log 2>&1

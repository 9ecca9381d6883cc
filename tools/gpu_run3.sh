#!/bin/bash
# new kernels: parity tests, then per-class profile + solver-parameter sweep on cfg2, cfg4 with the best
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu3.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu3.log
for a in "--eta 0" "--eta 0.01" "--eta 0.1" "--eta 0.01 --nu 3" "--eta 0.01 --kmode 1" "--eta 0.01 --omega 0.8"; do
  echo "=== cfg2 $a" >> $O/sweep3_cfg2.log
  timeout 300 python tools/probe.py --cfg 2 --steps 1 --profile $a >> $O/sweep3_cfg2.log 2>&1
done
timeout 300 python tools/probe.py --cfg 1 --steps 2 --profile --eta 0.01 > $O/probe3_cfg1.log 2>&1
timeout 300 python tools/probe.py --cfg 3 --steps 1 --profile --eta 0.01 > $O/probe3_cfg3.log 2>&1
timeout 900 python tools/probe.py --cfg 4 --steps 1 --profile --eta 0.01 > $O/probe3_cfg4.log 2>&1

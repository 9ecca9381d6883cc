#!/bin/bash
# stored diagonal for the smoother: bit identity + timing of the V-cycle and the step at cfg4
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build41.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "diagonal or deep" > $O/pytest_gpu41a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu41a.log
for c in 4 2; do
  for d in 0 1; do
    echo "=== cfg$c HJB_NO_DIAG=$d" >> $O/opbench41.log
    if [ $d = 1 ]; then export HJB_NO_DIAG=1; else unset HJB_NO_DIAG; fi
    timeout 400 python tools/opbench.py --cfg $c --reps 8 --only vcycle >> $O/opbench41.log 2>&1
  done
done
unset HJB_NO_DIAG
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --json-out $O/bench41_cfg4.json > $O/bench41_cfg4.log 2>&1

#!/bin/bash
# window search over the whole interior (general geometry) vs deep box only vs direct
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build36.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu36a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu36a.log
for c in 3 2 1 4; do
  for w in 2 1 0; do
    echo "=== cfg$c HJB_WIN=$w" >> $O/opbench36.log
    HJB_WIN=$w timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench36.log 2>&1
  done
done
for c in 3 2; do
  timeout 600 python bench.py --config cfg$c --no-cpu-baseline --json-out $O/bench36_cfg$c.json > $O/bench36_cfg$c.log 2>&1
done

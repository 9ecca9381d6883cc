#!/bin/bash
# timing threshold 16384 nodes: smoke, bench cfg1-4 (+ untimed cfg4/cfg2), all GPU tests
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build53.log 2>&1; echo "build exit $?" >> $O/build53.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $O/smoke53.log 2>&1; echo "smoke exit $?" >> $O/smoke53.log
timeout 1200 python bench.py --json-out $O/bench53_cfg4.json > $O/bench53_cfg4.log 2>&1; echo "exit $?" >> $O/bench53_cfg4.log
for c in 3 2 1; do
  timeout 600 python bench.py --config cfg$c --json-out $O/bench53_cfg$c.json > $O/bench53_cfg$c.log 2>&1; echo "exit $?" >> $O/bench53_cfg$c.log
done
for c in cfg4 cfg2; do
  timeout 900 python bench.py --config $c --no-time-kernels --no-cpu-baseline --no-e2e --json-out $O/bench53_${c}_notime.json > $O/bench53_${c}_notime.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu53.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu53.log

#!/bin/bash
# new defaults (window search, general search at 168 registers): smoke, all GPU tests, bench cfg1-4
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build38.log 2>&1; echo "build exit $?" >> $O/build38.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $O/smoke38.log 2>&1; echo "smoke exit $?" >> $O/smoke38.log
timeout 1200 python bench.py --json-out $O/bench38_cfg4.json > $O/bench38_cfg4.log 2>&1; echo "exit $?" >> $O/bench38_cfg4.log
for c in 3 2 1; do
  timeout 600 python bench.py --config cfg$c --json-out $O/bench38_cfg$c.json > $O/bench38_cfg$c.log 2>&1; echo "exit $?" >> $O/bench38_cfg$c.log
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu38.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu38.log

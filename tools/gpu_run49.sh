#!/bin/bash
# event-timing ring (no pipeline drains): bench cfg1-4 with and without per-kernel timing, all GPU tests
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build49.log 2>&1; echo "build exit $?" >> $O/build49.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $O/smoke49.log 2>&1; echo "smoke exit $?" >> $O/smoke49.log
timeout 1200 python bench.py --json-out $O/bench49_cfg4.json > $O/bench49_cfg4.log 2>&1; echo "exit $?" >> $O/bench49_cfg4.log
timeout 1200 python bench.py --no-time-kernels --no-cpu-baseline --no-e2e --json-out $O/bench49_cfg4_notime.json > $O/bench49_cfg4_notime.log 2>&1
for c in 3 2 1; do
  timeout 600 python bench.py --config cfg$c --json-out $O/bench49_cfg$c.json > $O/bench49_cfg$c.log 2>&1; echo "exit $?" >> $O/bench49_cfg$c.log
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu49.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu49.log

#!/bin/bash
# defaults with the W-cycle: smoke, bench cfg1-4 (+ cfg4 without per-kernel event timing)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build48.log 2>&1; echo "build exit $?" >> $O/build48.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $O/smoke48.log 2>&1; echo "smoke exit $?" >> $O/smoke48.log
timeout 1200 python bench.py --json-out $O/bench48_cfg4.json > $O/bench48_cfg4.log 2>&1; echo "exit $?" >> $O/bench48_cfg4.log
timeout 1200 python bench.py --no-time-kernels --no-cpu-baseline --no-e2e --json-out $O/bench48_cfg4_notime.json > $O/bench48_cfg4_notime.log 2>&1
for c in 3 2 1; do
  timeout 600 python bench.py --config cfg$c --json-out $O/bench48_cfg$c.json > $O/bench48_cfg$c.log 2>&1; echo "exit $?" >> $O/bench48_cfg$c.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench48_ref.log 2>&1; echo "exit $?" >> $O/bench48_ref.log

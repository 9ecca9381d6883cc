#!/bin/bash
# stored-diagonal smoother as default: all GPU tests, bench cfg1-4, ncu of one cfg4 V-cycle
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build42.log 2>&1; echo "build exit $?" >> $O/build42.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $O/smoke42.log 2>&1; echo "smoke exit $?" >> $O/smoke42.log
timeout 1200 python bench.py --json-out $O/bench42_cfg4.json > $O/bench42_cfg4.log 2>&1; echo "exit $?" >> $O/bench42_cfg4.log
for c in 3 2 1; do
  timeout 600 python bench.py --config cfg$c --json-out $O/bench42_cfg$c.json > $O/bench42_cfg$c.log 2>&1; echo "exit $?" >> $O/bench42_cfg$c.log
done
CMD="python tools/opbench.py --cfg 4 --reps 2 --only vcycle"
timeout 600 $CMD > $O/plain42.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator|k_jacobi0" -s 0 -c 15 -o $O/prof42_cfg4 $CMD > $O/ncu42.log 2>&1
echo "ncu exit $?" >> $O/ncu42.log
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu42.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu42.log

#!/bin/bash
# consolidated check of the current defaults: build, smoke, all GPU tests, bench cfg4/3/2/1,
# gather cache-operator variants, launch list of one cfg4 step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build31.log 2>&1; echo "build exit $?" >> $O/build31.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print('smoke ok')" > $O/smoke31.log 2>&1; echo "smoke exit $?" >> $O/smoke31.log
timeout 1200 python bench.py --json-out $O/bench31_cfg4.json > $O/bench31_cfg4.log 2>&1; echo "exit $?" >> $O/bench31_cfg4.log
for c in 3 2 1; do
  timeout 600 python bench.py --config cfg$c --json-out $O/bench31_cfg$c.json > $O/bench31_cfg$c.log 2>&1; echo "exit $?" >> $O/bench31_cfg$c.log
done
for v in gld0 gld1 gld2; do
  echo "=== $v" >> $O/opbench31.log
  HJB_LIB=build_variants/$v.so timeout 400 python tools/opbench.py --cfg 4 --reps 6 >> $O/opbench31.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu31.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu31.log

#!/bin/bash
# deep + strips (TMA opt-in): tests, default bench, ncu full capture of the deep Jacobi + apply
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build19.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu19.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu19.log
timeout 1200 python bench.py --json-out $O/bench19_cfg4.json > $O/bench19_cfg4.log 2>&1; echo "exit $?" >> $O/bench19_cfg4.log
CMD="python tools/opbench.py --cfg 4 --reps 2 --only apply,vcycle"
timeout 600 $CMD > $O/plain19.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator" -s 10 -c 12 -o $O/prof19_cfg4 $CMD > $O/ncu19.log 2>&1
echo "ncu exit $?" >> $O/ncu19.log

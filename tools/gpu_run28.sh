#!/bin/bash
# current defaults: all GPU tests, default bench (cfg4), cfg2/cfg3 bench lines, ncu of the deep Jacobi + search
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build28.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu28.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu28.log
timeout 1200 python bench.py --json-out $O/bench28_cfg4.json > $O/bench28_cfg4.log 2>&1; echo "exit $?" >> $O/bench28_cfg4.log
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --json-out $O/bench28_cfg2.json > $O/bench28_cfg2.log 2>&1
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --json-out $O/bench28_cfg3.json > $O/bench28_cfg3.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --json-out $O/bench28_cfg1.json > $O/bench28_cfg1.log 2>&1
CMD="python tools/opbench.py --cfg 4 --reps 2"
timeout 600 $CMD > $O/plain28.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator|k_search" -s 12 -c 14 -o $O/prof28_cfg4 $CMD > $O/ncu28.log 2>&1
echo "ncu exit $?" >> $O/ncu28.log

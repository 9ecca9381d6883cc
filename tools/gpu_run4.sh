#!/bin/bash
# slabs (thread ranks) + all GPU tests; kernel-level timing cfg4/cfg2; ncu full capture of the fine apply (cfg4)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build4.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu4.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu4.log
timeout 600 python tools/opbench.py --cfg 4 --reps 10 > $O/opbench4_cfg4.log 2>&1; echo "exit $?" >> $O/opbench4_cfg4.log
timeout 300 python tools/opbench.py --cfg 2 --reps 20 > $O/opbench4_cfg2.log 2>&1; echo "exit $?" >> $O/opbench4_cfg2.log
CMD="python tools/opbench.py --cfg 4 --reps 2 --only apply"
timeout 600 $CMD > $O/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_operator -s 2 -c 1 -o $O/prof4_apply_cfg4 $CMD > $O/ncu4.log 2>&1
echo "ncu exit $?" >> $O/ncu4.log

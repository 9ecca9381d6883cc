#!/bin/bash
# new defaults: bench cfg4 (default command), ncu launch list of one cfg4 step, ncu full of apply + search
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build13.log 2>&1
timeout 1200 python bench.py --json-out $O/bench13_cfg4.json > $O/bench13_cfg4.log 2>&1; echo "exit $?" >> $O/bench13_cfg4.log
CMD="python tools/opbench.py --cfg 4 --reps 2"
timeout 600 $CMD > $O/plain13.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator|k_search" -s 2 -c 4 -o $O/prof13_cfg4 $CMD > $O/ncu13.log 2>&1
echo "ncu exit $?" >> $O/ncu13.log
CMD2="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-time-kernels"
timeout 900 $CMD2 > $O/plain13b.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $O/launches13_cfg4.csv $CMD2 > $O/ncu13b.log 2>&1
echo "ncu exit $?" >> $O/ncu13b.log

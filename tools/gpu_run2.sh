#!/bin/bash
# bench + fp64 peak + ncu launch list and one full capture (cfg2) -- round 1, first measured path
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out
mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu && ./tools/fp64_peak > $O/fp64_peak.json 2>&1
timeout 600 python bench.py --config cfg2 --steps 3 --warmup 3 --json-out $O/bench_cfg2.json > $O/bench_cfg2.log 2>&1; echo "exit $?" >> $O/bench_cfg2.log
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --json-out $O/bench_cfg4.json > $O/bench_cfg4.log 2>&1; echo "exit $?" >> $O/bench_cfg4.log
CMD="python bench.py --config cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-time-kernels"
timeout 300 $CMD > $O/plain_cfg2.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file $O/launches_cfg2.csv $CMD > $O/ncu_launch_cfg2.log 2>&1
echo "launches exit $?" >> $O/ncu_launch_cfg2.log
timeout 300 $CMD > $O/plain_cfg2b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_operator -s 200 -c 3 -o $O/prof_op_cfg2 $CMD > $O/ncu_full_cfg2.log 2>&1
echo "full exit $?" >> $O/ncu_full_cfg2.log

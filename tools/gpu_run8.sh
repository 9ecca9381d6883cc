#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q > $O/pytest_gpu8.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu8.log
timeout 1200 python bench.py --steps 3 --warmup 3 --json-out $O/bench8_cfg4.json > $O/bench8_cfg4.log 2>&1; echo "exit $?" >> $O/bench8_cfg4.log
timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench8_cfg2.json > $O/bench8_cfg2.log 2>&1; echo "exit $?" >> $O/bench8_cfg2.log
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench8_cfg3.json > $O/bench8_cfg3.log 2>&1; echo "exit $?" >> $O/bench8_cfg3.log

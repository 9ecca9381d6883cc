#!/bin/bash
# strip launches for the boundary layer; TMA alignment fix; A/B deep/tma on the full step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build18.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu18a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu18a.log
for m in "HJB_NO_DEEP=1" "HJB_NO_TMA=1" "HJB_X=0"; do
  echo "=== [$m]" >> $O/opbench18.log
  env $m timeout 300 python tools/opbench.py --cfg 4 --reps 6 >> $O/opbench18.log 2>&1
  echo "=== bench [$m]" >> $O/ab18.log
  env $m timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline >> $O/ab18.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu18.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu18.log

#!/bin/bash
# deep search kernel; correctness; smoothing-sweep / forcing sweep at cfg4 (bench)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build15.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu15a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu15a.log
for c in 4 2; do
  echo "=== cfg$c deep" >> $O/opbench15.log
  timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench15.log 2>&1
  echo "=== cfg$c general" >> $O/opbench15.log
  HJB_NO_DEEP=1 timeout 300 python tools/opbench.py --cfg $c --reps 10 --only search >> $O/opbench15.log 2>&1
done
for a in "--nu 1" "--nu 2" "--nu 3" "--nu 2 --pi-forcing 0.3" "--nu 2 --pi-forcing 0.03"; do
  echo "=== $a" >> $O/sweep15.log
  timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline $a >> $O/sweep15.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu15.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu15.log

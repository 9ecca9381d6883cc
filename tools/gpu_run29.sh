#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build29.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > $O/pytest_gpu29.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu29.log
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline --json-out $O/bench29_cfg3.json > $O/bench29_cfg3.log 2>&1
for a in "--nu 1" "--nu 3" "--pi-forcing 0.03" "--pi-forcing 0.3" "--nu 3 --pi-forcing 0.03"; do
  echo "=== $a" >> $O/sweep29.log
  timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline $a >> $O/sweep29.log 2>&1
done
CMD="python tools/opbench.py --cfg 4 --reps 2 --only vcycle"
timeout 600 $CMD > $O/plain29.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator" -s 0 -c 8 -o $O/prof29_cfg4 $CMD > $O/ncu29.log 2>&1
echo "ncu exit $?" >> $O/ncu29.log

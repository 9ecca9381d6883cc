#!/bin/bash
# W-cycle on the large levels as the library default: thresholds, then all GPU tests
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build46.log 2>&1
for c in cfg4 cfg2; do
  for t in 65536 131072 262144; do
    echo "=== $c gamma_min=$t" >> $O/sweep46.log
    if [ $c = cfg4 ]; then S="--steps 3 --warmup 3"; else S="--steps 8 --warmup 3"; fi
    timeout 600 python bench.py --config $c $S --no-e2e --no-cpu-baseline --gamma-min $t >> $O/sweep46.log 2>&1
  done
done
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu46.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu46.log

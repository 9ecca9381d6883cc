#!/bin/bash
# cycle index 3 on the largest levels; revisit threshold with forcing 0.01 (untimed step times)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for a in "--gamma 2" "--gamma 3" "--gamma 3 --gamma-min 1000000" "--gamma 2 --gamma-min 262144"; do
  for c in cfg4 cfg2; do
    echo "=== $c $a" >> $O/sweep54.log
    if [ $c = cfg4 ]; then S="--steps 3 --warmup 3"; else S="--steps 8 --warmup 3"; fi
    timeout 600 python bench.py --config $c $S --no-e2e --no-cpu-baseline --no-time-kernels $a >> $O/sweep54.log 2>&1
  done
done

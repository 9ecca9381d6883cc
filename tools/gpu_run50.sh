#!/bin/bash
# forcing term with the W-cycle (solves are cheap now, the search dominates): PI count vs step time
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for c in cfg4 cfg2; do
  for e in 0.0 0.003 0.01 0.03 0.1; do
    echo "=== $c pi_forcing=$e" >> $O/sweep50.log
    if [ $c = cfg4 ]; then S="--steps 3 --warmup 3"; else S="--steps 8 --warmup 3"; fi
    timeout 600 python bench.py --config $c $S --no-e2e --no-cpu-baseline --no-time-kernels --pi-forcing $e >> $O/sweep50.log 2>&1
  done
done

#!/bin/bash
# solver settings at cfg4: V(nu1,nu2) asymmetric cycles, smaller forcing
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
for a in "" "--nu-pre 1 --nu-post 2" "--nu-pre 2 --nu-post 1" "--nu-pre 1 --nu-post 3" "--pi-forcing 0.01" "--pi-forcing 0.003" "--nu-pre 1 --nu-post 2 --pi-forcing 0.01"; do
  echo "=== $a" >> $O/sweep40.log
  timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $a >> $O/sweep40.log 2>&1
done

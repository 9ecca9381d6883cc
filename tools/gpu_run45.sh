#!/bin/bash
# W-cycle restricted to large coarse levels (HJB_MG_GAMMA_MIN owned nodes): step time per config
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build45.log 2>&1
for c in cfg4 cfg2 cfg3 cfg1; do
  for t in none 0 4096 16384 65536 262144; do
    if [ $t = none ]; then E=""; else E="HJB_MG_GAMMA=2 HJB_MG_GAMMA_MIN=$t"; fi
    echo "=== $c [$E]" >> $O/sweep45.log
    if [ $c = cfg4 ]; then S="--steps 2 --warmup 3"; else S="--steps 5 --warmup 3"; fi
    env $E timeout 600 python bench.py --config $c $S --no-e2e --no-cpu-baseline >> $O/sweep45.log 2>&1
  done
done

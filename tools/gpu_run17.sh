#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build17.log 2>&1
HJB_NO_TMA=1 timeout 120 python tools/debug_deep.py 1 > $O/debug17.log 2>&1
HJB_NO_TMA=1 timeout 120 python tools/debug_deep.py 2 >> $O/debug17.log 2>&1
for m in "" "HJB_NO_DEEP=1"; do
  echo "=== [$m]" >> $O/ab17.log
  env $m HJB_NO_TMA=1 timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline >> $O/ab17.log 2>&1
done

#!/bin/bash
# cycle index (W-cycle) and extra coarse-level smoothing: V-cycle contraction, BiCGSTAB its, step time
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build44.log 2>&1
for e in "" "HJB_MG_GAMMA=2" "HJB_NU_COARSE=4" "HJB_MG_GAMMA=2 HJB_NU_COARSE=3"; do
  for c in "4 --m 30" 2; do
    echo "=== cfg$c [$e]" >> $O/kry44.log
    env $e timeout 400 python tools/krylov_study.py --cfg $c --no-gmres --exact-only >> $O/kry44.log 2>&1
  done
  echo "=== [$e]" >> $O/sweep44.log
  env $e timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline >> $O/sweep44.log 2>&1
done

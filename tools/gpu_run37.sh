#!/bin/bash
# window search variants (threads x control split x unroll), deep-box and whole-interior modes
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build37.log 2>&1
for c in 3 2; do
  for v in default w512s4 w512s2u2 w256s1; do
    for w in 2 1; do
      echo "=== cfg$c $v HJB_WIN=$w" >> $O/opbench37.log
      if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
      HJB_LIB=$L HJB_WIN=$w timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench37.log 2>&1
    done
  done
done

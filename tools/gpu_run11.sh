#!/bin/bash
# workload sensitivity of the operator kernel (noise fields, policy variability) + ncu of cfg4 apply
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build11.log 2>&1
for a in "--cfg 4" "--cfg 4 --policy zero" "--cfg 4 --policy random" "--cfg 1 --n 16385" "--cfg 1 --n 16385 --policy zero" "--cfg 2" "--cfg 1 --n 4097"; do
  echo "=== $a" >> $O/opbench11.log
  timeout 300 python tools/opbench.py $a --reps 6 --only apply >> $O/opbench11.log 2>&1
done
CMD="python tools/opbench.py --cfg 4 --reps 2 --only apply,vcycle"
timeout 600 $CMD > $O/plain11.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_operator -s 2 -c 4 -o $O/prof11_cfg4 $CMD > $O/ncu11.log 2>&1
echo "ncu exit $?" >> $O/ncu11.log

#!/bin/bash
# occupancy of the general (boundary-strip) search kernel; launch split of the cfg3 search
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build35.log 2>&1
for c in 3 2 4; do
  echo "=== cfg$c default" >> $O/opbench35.log
  timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench35.log 2>&1
  for v in s_minb2 s_minb3 s_minb4; do
    echo "=== cfg$c $v" >> $O/opbench35.log
    HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench35.log 2>&1
  done
done
CMD="python tools/opbench.py --cfg 3 --reps 10 --only search"
timeout 300 $CMD > $O/plain35.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches35_cfg3.csv $CMD > $O/ncu35.log 2>&1
echo "ncu exit $?" >> $O/ncu35.log

#!/bin/bash
# Krylov study (BiCGSTAB vs GMRES prototype, V-cycle contraction, MG knobs) + ncu of the fine Jacobi
# sweep at cfg4 + launch list of one cfg4 step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build32.log 2>&1
for a in "--cfg 2" "--cfg 2 --kmode 1" "--cfg 2 --omega 0.8" "--cfg 2 --omega 0.6" "--cfg 2 --nu 3" "--cfg 1" "--cfg 3" "--cfg 4 --m 30"; do
  echo "=== $a" >> $O/krylov32.log
  timeout 600 python tools/krylov_study.py $a >> $O/krylov32.log 2>&1
done
CMD="python tools/opbench.py --cfg 4 --reps 2 --only vcycle"
timeout 600 $CMD > $O/plain32.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_operator" -s 0 -c 15 -o $O/prof32_cfg4 $CMD > $O/ncu32.log 2>&1
echo "ncu exit $?" >> $O/ncu32.log
CMD2="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-time-kernels"
timeout 900 $CMD2 > $O/plain32b.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches32_cfg4.csv $CMD2 > $O/ncu32b.log 2>&1
echo "ncu exit $?" >> $O/ncu32b.log

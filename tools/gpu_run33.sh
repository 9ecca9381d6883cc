#!/bin/bash
# shared-memory window search: bit identity, timing vs the direct deep kernel, thread-count variants
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build33.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu33a.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu33a.log
for c in 3 2 1; do
  echo "=== cfg$c win" >> $O/opbench33.log
  timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench33.log 2>&1
  echo "=== cfg$c direct" >> $O/opbench33.log
  HJB_WIN=0 timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench33.log 2>&1
done
for v in win384 win512; do
  for c in 3 2; do
    echo "=== cfg$c $v" >> $O/opbench33.log
    HJB_LIB=build_variants/$v.so timeout 300 python tools/opbench.py --cfg $c --reps 20 --only search >> $O/opbench33.log 2>&1
  done
done
for c in 3 2; do
  timeout 600 python bench.py --config cfg$c --no-cpu-baseline --json-out $O/bench33_cfg$c.json > $O/bench33_cfg$c.log 2>&1
done
# coarse-level SL step rule (coarse_k_mode 2 with factors A, B): V-cycle contraction + BiCGSTAB its
for c in "4 --m 30" 2 1 3; do
  for v in kc_a05b1 kc_a1b1 kc_a2b1 kc_a1b05 kc_a2b2; do
    echo "=== cfg$c $v kmode2" >> $O/kc33.log
    HJB_LIB=build_variants/$v.so timeout 300 python tools/krylov_study.py --cfg $c --kmode 2 --no-gmres --exact-only >> $O/kc33.log 2>&1
  done
  echo "=== cfg$c kmode0" >> $O/kc33.log
  timeout 300 python tools/krylov_study.py --cfg $c --no-gmres --exact-only >> $O/kc33.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest_gpu33.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu33.log

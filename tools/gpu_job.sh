#!/bin/bash
# tools/gpu_job.sh JOB [ARGS...] -- the GPU-side jobs of this repo, run on a gpurun box from the repo
# root (one parameterised driver instead of one-off scripts).  Outputs go to gpurun_out/<tag>*.
#   build                       build libhjb.so + the C certificate oracle
#   tests [PYTEST_ARGS...]      pytest -m gpu (durations, log in gpurun_out/pytest_<tag>.log)
#   bench TAG CFG [ARGS...]     python bench.py --config CFG [ARGS] -> gpurun_out/bench_<TAG>_<CFG>.json
#   launches TAG CMD...         plain run of CMD, then the ncu launch list (gpu__time_duration per launch)
#   ncufull TAG REGEX SKIP CMD... plain run of CMD, then ncu --set full of COUNT=2 launches matching REGEX
#   opbench TAG CFG [ARGS...]   tools/opbench.py kernel timings
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
job=$1; shift
TAG=${TAG:-run}
case $job in
  build)
    python -c "import paper_1605_04821_b200.build as b; b.build(force=True)" > $O/build_$TAG.log 2>&1
    python -c "from oracle import certify; certify.build(force=True)" >> $O/build_$TAG.log 2>&1 ;;
  tests)
    timeout ${TIMEOUT:-1500} python -m pytest tests -m gpu -q -rA --durations=30 "$@" > $O/pytest_$TAG.log 2>&1
    echo "pytest rc=$?" >> $O/pytest_$TAG.log ;;
  bench)
    tag=$1; cfg=$2; shift 2
    timeout ${TIMEOUT:-900} python bench.py --config $cfg --json-out $O/bench_${tag}_$cfg.json "$@" > $O/bench_${tag}_$cfg.log 2>&1
    echo "bench rc=$?" >> $O/bench_${tag}_$cfg.log ;;
  launches)
    tag=$1; shift
    timeout 600 "$@" > $O/plain_$tag.log 2>&1 && \
      timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$tag.csv "$@" > $O/ncu_$tag.log 2>&1
    echo "ncu rc=$?" >> $O/ncu_$tag.log ;;
  ncufull)
    tag=$1; re=$2; skip=$3; shift 3
    timeout 600 "$@" > $O/plain_$tag.log 2>&1 && \
      timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c ${COUNT:-2} \
        -o $O/prof_$tag "$@" > $O/ncu_$tag.log 2>&1
    echo "ncu rc=$?" >> $O/ncu_$tag.log ;;
  opbench)
    tag=$1; cfg=$2; shift 2
    timeout 600 python tools/opbench.py --cfg $cfg "$@" > $O/opbench_${tag}_$cfg.log 2>&1 ;;
  *) echo "unknown job $job"; exit 2 ;;
esac

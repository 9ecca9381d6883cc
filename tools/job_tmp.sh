cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "nested" > $O/q_pytest.log 2>&1; echo "rc=$?" >> $O/q_pytest.log
for u in 1 3 8; do
timeout 900 python bench.py --config cfg4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-time-kernels --nested-upto $u --nested-increment 1 --json-out $O/q_bench_inc$u.json > $O/q_bench_inc$u.log 2>&1
done

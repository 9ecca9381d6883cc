cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "nested or deep_kernels" > $O/j4_pytest.log 2>&1; echo "rc=$?" >> $O/j4_pytest.log
timeout 900 python bench.py --config cfg4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --nested-upto 1 --json-out $O/j4_bench_n1.json > $O/j4_bench_n1.log 2>&1
timeout 900 python bench.py --config cfg4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --nested-upto 3 --json-out $O/j4_bench_n3.json > $O/j4_bench_n3.log 2>&1
timeout 900 python bench.py --config cfg4 --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --nested-upto 8 --json-out $O/j4_bench_n8.json > $O/j4_bench_n8.log 2>&1

cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "deep_kernels or fullsize or step_parity or slab or nested or certificate" > $O/w_pytest.log 2>&1; echo "rc=$?" >> $O/w_pytest.log
timeout 300 python tools/opbench.py --cfg 4 --only search,apply,vcycle --reps 20 > $O/w_opbench.log 2>&1
timeout 1200 python bench.py --config cfg4 --steps 16 --warmup 3 --stats-jsonl $O/w_stats_cfg4.jsonl --json-out $O/w_bench_cfg4.json > $O/w_bench_cfg4.log 2>&1

cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "stalled or deep_kernels or agmg or slab_apply" > $O/s_pytest.log 2>&1; echo "rc=$?" >> $O/s_pytest.log
timeout 600 python bench.py --config cfg3 --steps 16 --warmup 3 --no-e2e --no-cpu-baseline --json-out $O/s_bench_cfg3.json > $O/s_bench_cfg3.log 2>&1
timeout 1500 python tools/paper_context.py > $O/s_paper_context.log 2>&1

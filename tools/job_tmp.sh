cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=20 > $O/r_pytest.log 2>&1; echo "rc=$?" >> $O/r_pytest.log
timeout 1200 python tools/paper_context.py > $O/r_paper_context.log 2>&1
timeout 600 python bench.py --config cfg2 --steps 16 --warmup 3 --no-e2e --json-out $O/r_bench_cfg2.json > $O/r_bench_cfg2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/r_smoke.log 2>&1

cd $GRAFT_REPO_ROOT
O=gpurun_out
TAG=fin bash tools/gpu_job.sh tests
python -c "import __graft_entry__ as g; g.smoke()" > $O/fin_smoke.log 2>&1
for c in cfg1 cfg2 cfg3; do
  timeout 900 python bench.py --config $c --steps 16 --warmup 3 --json-out $O/fin_bench_$c.json > $O/fin_bench_$c.log 2>&1
done
timeout 1500 python bench.py --config cfg4 --steps 16 --warmup 3 --stats-jsonl $O/fin_stats_cfg4.jsonl --json-out $O/fin_bench_cfg4.json > $O/fin_bench_cfg4.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/fin_launches_cfg4.csv python bench.py --config cfg4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-time-kernels > $O/fin_ncu_launches.log 2>&1
COUNT=1 bash tools/gpu_job.sh ncufull fin_search "k_search_deep2" 5 python tools/opbench.py --cfg 4 --only search --reps 10

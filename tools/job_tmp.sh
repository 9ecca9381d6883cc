cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "agmg or stalled or deep_kernels or slab or galerkin or step_parity" > $O/u_pytest.log 2>&1; echo "rc=$?" >> $O/u_pytest.log
timeout 1500 python tools/paper_context.py > $O/u_paper_context.log 2>&1
timeout 900 python tools/agmg_study.py --cfg 2 --steps 3 > $O/u_agmg_cfg2.log 2>&1
timeout 600 python tools/agmg_study.py --cfg 1 --steps 3 > $O/u_agmg_cfg1.log 2>&1
timeout 600 python tools/opbench.py --cfg 4 --only vcycle --reps 20 > $O/u_opbench_vcycle.log 2>&1

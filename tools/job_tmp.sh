cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/opbench.py --cfg 4 --only search --reps 30 > $O/j7_opbench_2p3.log 2>&1
HJB_LIB=build_variants/s2p4.so timeout 300 python tools/opbench.py --cfg 4 --only search --reps 30 > $O/j7_opbench_2p4.log 2>&1
HJB_NO_SEARCH2P=1 timeout 300 python tools/opbench.py --cfg 4 --only search --reps 30 > $O/j7_opbench_deep2.log 2>&1
timeout 300 python tools/opbench.py --cfg 2 --only search --reps 30 > $O/j7_opbench_2p3_cfg2.log 2>&1
HJB_NO_SEARCH2P=1 timeout 300 python tools/opbench.py --cfg 2 --only search --reps 30 > $O/j7_opbench_deep2_cfg2.log 2>&1

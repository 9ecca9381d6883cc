#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test tools/tma_test.cu > $O/tma20.log 2>&1
timeout 60 ./tools/tma_test >> $O/tma20.log 2>&1; echo "exit $?" >> $O/tma20.log
python -c "import paper_1605_04821_b200.build as b; b.build()" > $O/build20.log 2>&1
HJB_TMA=1 timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "deep" > $O/pytest_gpu20.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu20.log
HJB_TMA=1 timeout 300 python tools/opbench.py --cfg 4 --reps 10 --only search >> $O/opbench20.log 2>&1
timeout 300 python tools/opbench.py --cfg 4 --reps 10 --only search >> $O/opbench20.log 2>&1

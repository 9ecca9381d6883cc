#!/bin/bash
# first GPU probe of the round: parity tests + iteration counts / timings per config
cd "$GRAFT_REPO_ROOT" || cd /root/repo
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in "1 --steps 2" "2 --steps 2" "3 --steps 1" "4 --steps 1"; do
  set -- $c
  timeout 600 python tools/probe.py --cfg $c > gpurun_out/probe_cfg$1.log 2>&1; echo "exit $?" >> gpurun_out/probe_cfg$1.log
done

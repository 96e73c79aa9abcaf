#!/bin/bash
# Session-4 call 1: rotation A/B (new vs pre-rotation tree in baseline/r2h), then the whole GPU suite and smoke at HEAD.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
bash tools/gpu_r02_rot.sh > $O/rot_ab.txt 2>&1; cat $O/rot_ab.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -4 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log

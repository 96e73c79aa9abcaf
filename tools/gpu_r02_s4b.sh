#!/bin/bash
# Session-4 call 2: the fixed quasi-optimality default and the KMAX-split rotation (targeted tests, rotation alone), then the final measurement script.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pl1.py tests/test_gpu_multirank.py tests/test_gpu_kernels.py tests/test_gpu_solve.py -q -rf --timeout 600 -k "quasi or pl1_loopback or rotate or solve" > $O/s4b_pytest.log 2>&1; echo "pytest rc=$?" >> $O/s4b_pytest.log; tail -3 $O/s4b_pytest.log
for a in "C5 24 10" "C5 16 10" "C3 32 20" "C3 48 20" "C2 30 12" "C2 24 12"; do
  timeout 300 python tools/rot_time.py $a 20 2>&1 | tail -1
done > $O/s4b_rot.txt 2>&1; cat $O/s4b_rot.txt
bash tools/gpu_final.sh

mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -rf --timeout 600 > $O/pytest_multirank.log 2>&1; echo "pytest rc=$?" >> $O/pytest_multirank.log
timeout 1200 bash tools/profile_round.sh C2 > gpurun_out/profile_C2.log 2>&1

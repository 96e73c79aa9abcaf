mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_pl1.py tests/test_gpu_multirank.py -m gpu -q -rf --timeout 300 > $O/pytest_pl1.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pl1.log

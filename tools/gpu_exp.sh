mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_solve.py -m gpu -q -rf --timeout 600 -k widest > $O/pytest_wide.log 2>&1; echo "pytest rc=$?" >> $O/pytest_wide.log

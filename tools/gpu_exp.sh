mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_pl1.py -m gpu -q -rf --timeout 300 -k wide > $O/pytest_pl1w.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pl1w.log

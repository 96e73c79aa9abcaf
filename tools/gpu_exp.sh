mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_reductions.py -m gpu -q -rf --timeout 300 > $O/pytest_red.log 2>&1; echo "rc=$?" >> $O/pytest_red.log

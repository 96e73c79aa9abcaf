mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_eig_tri.py -m gpu -q -rf --timeout 600 > $O/pytest_tri.log 2>&1; echo "rc=$?" >> $O/pytest_tri.log

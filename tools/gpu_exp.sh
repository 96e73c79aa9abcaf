mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_solve.py -m gpu -q -rf --timeout 300 -k graph_cache > $O/pytest_gc.log 2>&1; echo "rc=$?" >> $O/pytest_gc.log

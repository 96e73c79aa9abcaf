mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_solve.py -m gpu -q -rf --timeout 300 -k "grid" > $O/pytest_grid.log 2>&1; echo "pytest rc=$?" >> $O/pytest_grid.log

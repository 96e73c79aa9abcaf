mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_solve.py -m gpu -q -rf --timeout 600 -k pinned > $O/pytest_pin.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pin.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err

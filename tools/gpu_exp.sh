mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 1500 python -m pytest tests -m gpu -q -x -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
Q="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 python bench.py --config C3 $Q > $O/b_C3_def.json 2>&1
timeout 900 python bench.py --config C4 $Q > $O/b_C4_def.json 2>&1

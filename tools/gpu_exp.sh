mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
Q="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py --config C1 $Q > $O/b_C1_def.json 2>&1
TRPLK_NO_SMALL=1 timeout 600 python bench.py --config C1 $Q > $O/b_C1_nosmall.json 2>&1

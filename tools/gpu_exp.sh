mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 1500 python -m pytest tests -m gpu -q -x -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
Q="--steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
for i in 1 2; do
timeout 600 python bench.py --config C2 $Q > $O/b_C2_def$i.json 2>&1
TRPLK_NO_COOP3=1 timeout 600 python bench.py --config C2 $Q > $O/b_C2_nocoop$i.json 2>&1
done

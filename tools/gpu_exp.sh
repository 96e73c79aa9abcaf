mkdir -p gpurun_out/exp
O=gpurun_out/exp
TRPLK_K1=pipe timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -m gpu -q -x -rf --timeout 900 > $O/pytest_pipe.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pipe.log
Q="--steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
for c in C2 C3; do
  TRPLK_K1=pipe timeout 600 python bench.py --config $c $Q > $O/b_${c}_pipe.json 2>&1
  timeout 600 python bench.py --config $c $Q > $O/b_${c}_def.json 2>&1
done
TRPLK_K1=pipe timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/b_C5_pipe.json 2>&1
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/b_C5_def.json 2>&1

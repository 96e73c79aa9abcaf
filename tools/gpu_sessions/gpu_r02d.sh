#!/bin/bash
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py tests/test_gpu_torchrun.py tests/test_gpu_branches.py -q -x -k "block or no_precond or torchrun or branches or natural or breakdown" > $O/r02d_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/r02d_pytest.log
for B in 1 2 3; do
  timeout 900 python bench.py --config C5 --block $B --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02d_bench_C5_b$B.json 2> $O/r02d_bench_C5_b$B.err; echo "bench C5 b$B rc=$?"
done
timeout 900 python bench.py --config C2 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/r02d_bench_C2.json 2> $O/r02d_bench_C2.err; echo "bench C2 rc=$?"

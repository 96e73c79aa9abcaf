#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "block" > $O/r02c_block.log 2>&1; echo "block rc=$?"; tail -3 $O/r02c_block.log
timeout 1800 python -m pytest tests -m gpu -q > $O/r02c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r02c_pytest_gpu.log
tail -12 $O/r02c_pytest_gpu.log
for C in C5 C3 C2; do
  timeout 900 python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02c_bench_$C.json 2> $O/r02c_bench_$C.err; echo "bench $C rc=$?"
done

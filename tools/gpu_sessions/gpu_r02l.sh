#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x -k "no_precond" > $O/r02l_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 $O/r02l_pytest.log | grep -v "^$" | tail -25
for C in C2 C3; do
  timeout 900 python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --precond ic0 > $O/r02l_bench_${C}_ic0.json 2> $O/r02l_bench_${C}_ic0.err; echo "$C ic0 rc=$?"; tail -2 $O/r02l_bench_${C}_ic0.err
done
timeout 1200 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --precond ic0 > $O/r02l_bench_C5_ic0.json 2> $O/r02l_bench_C5_ic0.err; echo "C5 ic0 rc=$?"; tail -2 $O/r02l_bench_C5_ic0.err

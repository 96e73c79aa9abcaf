#!/bin/bash
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_solve.py -q -x -k "no_precond" > $O/r02m_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02m_pytest.log
timeout 300 python bench.py --config C2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --precond ic0 > $O/r02m_bench_C2_ic0.json 2> $O/r02m_bench_C2_ic0.err; echo "C2 ic0 rc=$?"
timeout 400 python bench.py --config C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --precond ic0 > $O/r02m_bench_C3_ic0.json 2> $O/r02m_bench_C3_ic0.err; echo "C3 ic0 rc=$?"
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --precond ic0 > $O/r02m_bench_C5_ic0.json 2> $O/r02m_bench_C5_ic0.err; echo "C5 ic0 rc=$?"

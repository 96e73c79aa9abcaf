#!/bin/bash
# DIA-C (constant diagonals) parity + C5/C3/C4/C2 lines; EIG=tri grid-path divergence probe.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py tests/test_gpu_multirank.py -q -x -m gpu > $O/r02o_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02o_pytest.log
TRPLK_EIG=tri timeout 300 python tools/cmp_traj.py 21 16 > $O/r02o_cmp_tri.log 2>&1; tail -8 $O/r02o_cmp_tri.log
timeout 300 python tools/cmp_traj.py 21 16 > $O/r02o_cmp_jac.log 2>&1; tail -4 $O/r02o_cmp_jac.log
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $O/r02o_bench_$c.json 2> $O/r02o_bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02o_bench_C5.json 2> $O/r02o_bench_C5.err; echo "C5 rc=$?"
TRPLK_DIAC=0 timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02o_bench_C5_nodiac.json 2> $O/r02o_bench_C5_nodiac.err; echo "C5 nodiac rc=$?"

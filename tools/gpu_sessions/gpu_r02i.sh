#!/bin/bash
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py tests/test_gpu_branches.py tests/test_gpu_multirank.py -q -x > $O/r02i_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/r02i_pytest.log
for P in 1 0; do
  TRPLK_PDL=$P timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/r02i_bench_C2_pdl$P.json 2> $O/r02i_bench_C2_pdl$P.err; echo "C2 pdl$P rc=$?"
  TRPLK_PDL=$P timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02i_bench_C3_pdl$P.json 2> $O/r02i_bench_C3_pdl$P.err; echo "C3 pdl$P rc=$?"
done

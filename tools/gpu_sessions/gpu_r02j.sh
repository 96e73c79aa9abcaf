#!/bin/bash
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -q -x -k "not C5" > $O/r02j_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/r02j_pytest.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02j_bench_C5.json 2> $O/r02j_bench_C5.err; echo "C5 rc=$?"
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --profile-last-only > $O/r02j_bench_C2.json 2> $O/r02j_bench_C2.err; echo "C2 rc=$?"
timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02j_bench_C3.json 2> $O/r02j_bench_C3.err; echo "C3 rc=$?"
python tools/c5_kernels.py 3 > $O/r02j_c5k.txt 2>&1

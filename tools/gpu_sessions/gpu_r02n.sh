#!/bin/bash
# Re-entry check of the round-2 tree: full GPU suite, smoke, driver-default bench (C5), C2/C3/C4 lines.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02n_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/r02n_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02n_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > $O/r02n_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/r02n_smoke.log
timeout 1200 python bench.py > $O/r02n_bench_default.json 2> $O/r02n_bench_default.err; echo "bench rc=$?"
for c in C2 C3 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/r02n_bench_$c.json 2> $O/r02n_bench_$c.err; echo "$c rc=$?"; done

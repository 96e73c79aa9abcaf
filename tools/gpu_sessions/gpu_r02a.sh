#!/bin/bash
# round-2 GPU check: host facts, full GPU suite, C5 bench (both arms)
O=gpurun_out
{ free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv; } > $O/r02_host.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r02_pytest_gpu.log
timeout 1200 python bench.py --steps 3 --warmup 2 > $O/r02_bench_C5.json 2> $O/r02_bench_C5.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/r02_ref_C5.json 2> $O/r02_ref_C5.err; echo "ref rc=$?"
tail -3 $O/r02_pytest_gpu.log

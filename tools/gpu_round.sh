# One gpurun call: GPU tests, default bench (full JSON line), per-config lines, profiles C2/C3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench rc=$?" >> gpurun_out/bench_C2.err
for c in C1 C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 1200 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 1200 bash tools/profile_round.sh C2 > gpurun_out/profile_C2.log 2>&1
timeout 1200 bash tools/profile_round.sh C3 > gpurun_out/profile_C3.log 2>&1

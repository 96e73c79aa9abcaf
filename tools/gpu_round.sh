# One gpurun call: GPU tests, default bench, variant comparisons, C3 bench, profiles.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench rc=$?" >> gpurun_out/bench_C2.err
Q="--steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
TRPLK_EIG=2b timeout 300 python bench.py $Q > gpurun_out/bench_C2_eig2b.json 2>&1
TRPLK_KVAR=rs timeout 300 python bench.py $Q > gpurun_out/bench_C2_rs.json 2>&1
timeout 900 python bench.py --config C3 $Q > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
TRPLK_KVAR=rs timeout 900 python bench.py --config C3 $Q > gpurun_out/bench_C3_rs.json 2>&1
timeout 1200 bash tools/profile_round.sh C2 > gpurun_out/profile_C2.log 2>&1

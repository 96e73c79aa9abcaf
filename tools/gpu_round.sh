# One gpurun call: default bench (full JSON), profiles of C2 and C3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench rc=$?" >> gpurun_out/bench_C2.err
timeout 1200 bash tools/profile_round.sh C2 > gpurun_out/profile_C2.log 2>&1
timeout 1200 bash tools/profile_round.sh C3 > gpurun_out/profile_C3.log 2>&1

mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 900 python -m pytest tests/test_gpu_pl1.py -m gpu -q -rf --timeout 300 > $O/pytest_pl1.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pl1.log
for c in C2 C3; do timeout 600 python bench.py --method pl1 --config $c > $O/bench_pl1_$c.json 2> $O/bench_pl1_$c.err; done

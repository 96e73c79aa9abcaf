mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 1500 python -m pytest tests -m gpu -q -x -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B2="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B2 > $O/plain2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file $O/launches_C2.csv $B2 > $O/ncu_l2.log 2>&1
python tools/ncu_summary.py launches $O/launches_C2.csv > $O/launches_C2_summary.txt 2>&1

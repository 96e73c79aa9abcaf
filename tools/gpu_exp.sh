mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 1500 python -m pytest tests -m gpu -q -x -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
Q="--steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
for c in C2 C3; do timeout 600 python bench.py --config $c $Q > $O/b_${c}_def.json 2>&1; done
B5="python bench.py --config C5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_rotate' -c 6 --csv --log-file $O/launches_C5rot.csv $B5 > $O/ncu_l5.log 2>&1
python tools/ncu_summary.py launches $O/launches_C5rot.csv > $O/launches_C5rot_summary.txt 2>&1

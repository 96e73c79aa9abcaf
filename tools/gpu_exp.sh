mkdir -p gpurun_out/exp
O=gpurun_out/exp
rm -f $O/sweep.txt
for i in 1 2; do
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(d['ms_per_step'], 'K1 us', round(r['ms_per_launch']*1e3,2), 'frac', r['frac'], 'inner us', round(r['inner_step']['ms']*1e3,2), r['inner_step']['share_ms'])" >> $O/sweep.txt
done
python tools/k1_scaling.py > $O/k1_scaling.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py -m gpu -q -x --timeout 300 > $O/pytest_spec.log 2>&1; echo "rc=$?" >> $O/pytest_spec.log

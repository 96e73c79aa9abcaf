mkdir -p gpurun_out/exp
O=gpurun_out/exp
rm -f $O/sweep.txt
for C in C2 C3 C2; do
echo "== $C" >> $O/sweep.txt
python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>>$O/sweep.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(d['ms_per_step'], d['config']['a_matvecs_per_solve'], 'K1 us', round(r['ms_per_launch']*1e3,2), 'frac', r['frac'], 'inner us', round(r['inner_step']['ms']*1e3,2), r['inner_step']['share_ms'])" >> $O/sweep.txt
done
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest_ks.log 2>&1; echo "rc=$?" >> $O/pytest_ks.log

mkdir -p gpurun_out/exp
O=gpurun_out/exp
rm -f $O/var.txt
for i in 1 2 3 4 5; do
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(d['ms_per_step'], d['value'], r['ms_per_launch']*1e3, r['frac'], d['clocks']['sm_mhz'])" >> $O/var.txt
done

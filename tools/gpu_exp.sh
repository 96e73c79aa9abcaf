mkdir -p gpurun_out/exp
O=gpurun_out/exp
for i in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_last.json 2>> $O/bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --profile-all-steps > $O/bench_all.json 2>> $O/bench.err
for f in bench_last bench_all; do python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', d['value'], d['ms_per_step'], r['achieved'], r['ms_per_launch'], r['samples'])" >> $O/prof_cmp.txt; done
done

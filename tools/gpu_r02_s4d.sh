#!/bin/bash
# Session-4 call 4: C2 / C3 at HEAD vs the round-1 final tree (baseline/r1, commit 05f8e5e) on the same box, alternating.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['solve']['a_matvecs_per_solve'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for i in 1 2 3; do
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C2 HEAD run $i"
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a2.json 2>/dev/null; pr /tmp/a2.json "C2 HEAD (profile on the last step only) run $i"
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/c.json 2>/dev/null); pr /tmp/c.json "C2 r1 run $i"
done > $O/s4d_ab.txt 2>&1
for i in 1 2; do
  timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C3 HEAD run $i"
  (cd baseline/r1 && timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/c.json 2>/dev/null); pr /tmp/c.json "C3 r1 run $i"
done >> $O/s4d_ab.txt 2>&1
cat $O/s4d_ab.txt

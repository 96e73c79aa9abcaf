#!/bin/bash
# After restoring r1's single DMMA chain in k_step1_rs2: C2 / C3 vs the round-1 tree, K1 alone.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json,sys;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for i in 1 2; do
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C2 main run $i"
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/c.json 2>/dev/null); pr /tmp/c.json "C2 r1 run $i"
done
timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C3 main"
for k in 15 23; do timeout 300 python tools/k1_time.py C2 $k 30 2>&1 | tail -1; done
timeout 300 python tools/k1_time.py C5 23 5 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/r02z_C2_launches.csv python tools/solve_twice.py C2 > /dev/null 2>&1
python tools/launch_sum.py $O/r02z_C2_launches.csv 2>&1 | head -14

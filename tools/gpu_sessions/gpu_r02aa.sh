#!/bin/bash
# mat_row without the DIA-C decode (experiment build) vs main vs round 1 at C2; K1 alone under ncu.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json,sys;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
X=$PWD/paper_1711_10128_b200/lib_exp/nodiacrow/libtrplk.so
for i in 1 2; do
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C2 main run $i"
  TRPLK_LIB_OVERRIDE=$X timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/b.json 2>/dev/null; pr /tmp/b.json "C2 nodiacrow run $i"
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/c.json 2>/dev/null); pr /tmp/c.json "C2 r1 run $i"
done
for L in main X; do
  if [ $L = X ]; then export TRPLK_LIB_OVERRIDE=$X; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_step1_rs2 --csv --log-file /tmp/k_$L.csv python tools/k1_time.py C2 23 20 > /dev/null 2>&1
  python tools/launch_sum.py /tmp/k_$L.csv 2>&1 | head -3 | sed "s/^/$L /"
done
unset TRPLK_LIB_OVERRIDE
(cd baseline/r1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_step1_rs2 --csv --log-file /tmp/k_r1.csv python tools/solve_twice.py C2 > /dev/null 2>&1); python tools/launch_sum.py /tmp/k_r1.csv 2>&1 | head -4 | sed "s/^/r1-solve /"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_step1_rs2 --csv --log-file /tmp/k_m2.csv python tools/solve_twice.py C2 > /dev/null 2>&1; python tools/launch_sum.py /tmp/k_m2.csv 2>&1 | head -4 | sed "s/^/main-solve /"

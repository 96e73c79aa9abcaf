#!/bin/bash
# C2 regression: current lib (mat_row DIA-C split) vs no-DUAL experiment build vs round-1 tree.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json,sys;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
NODUAL=$PWD/paper_1711_10128_b200/lib_exp/nodual/libtrplk.so
for i in 1 2; do
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C2 main run $i"
  TRPLK_LIB_OVERRIDE=$NODUAL timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/b.json 2>/dev/null; pr /tmp/b.json "C2 nodual run $i"
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/c.json 2>/dev/null); pr /tmp/c.json "C2 r1 run $i"
done
for k in 15 23; do
  timeout 300 python tools/k1_time.py C2 $k 30 2>&1 | tail -1
  TRPLK_LIB_OVERRIDE=$NODUAL timeout 300 python tools/k1_time.py C2 $k 30 2>&1 | tail -1 | sed 's/^/nodual /'
done
timeout 300 python tools/k1_time.py C5 15 5 2>&1 | tail -1
TRPLK_LIB_OVERRIDE=$NODUAL timeout 300 python tools/k1_time.py C5 23 5 2>&1 | tail -1 | sed 's/^/nodual /'
timeout 300 python tools/k1_time.py C5 23 5 2>&1 | tail -1

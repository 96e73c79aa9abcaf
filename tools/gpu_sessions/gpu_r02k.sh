#!/bin/bash
O=gpurun_out
REF=$PWD/paper_1711_10128_b200/lib_ref/libtrplk.so
for i in 1 2; do
  TRPLK_LIB_OVERRIDE=$REF timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02k_C5_ref$i.json 2>/dev/null
  timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02k_C5_new$i.json 2>/dev/null
done
for v in ref new; do for i in 1 2; do python -c "
import json;d=json.load(open('$O/r02k_C5_$v$i.json'));r=d['roofline'];print('$v$i',d['value'],round(d['ms_per_step']),r['frac'],r['inner_step']['frac'],d['clocks']['sm_mhz'],r['ms_per_launch'])"; done; done

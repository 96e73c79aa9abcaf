#!/bin/bash
# PDL on/off at C2 / C3 (process-level switch), alternating runs.
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do
  for p in 0 1; do
    TRPLK_PDL=$p timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > $O/r02u_C2_pdl$p.$i.json 2>/dev/null
    python -c "import json;d=json.load(open('$O/r02u_C2_pdl$p.$i.json'));print('C2 PDL=$p run $i', d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
for i in 1 2; do
  for p in 0 1; do
    TRPLK_PDL=$p timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --profile-last-only > $O/r02u_C3_pdl$p.$i.json 2>/dev/null
    python -c "import json;d=json.load(open('$O/r02u_C3_pdl$p.$i.json'));print('C3 PDL=$p run $i', d['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done

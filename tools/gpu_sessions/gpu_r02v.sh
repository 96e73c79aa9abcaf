#!/bin/bash
# Round-1 final tree (baseline/r1, commit 05f8e5e) vs the current tree, C2 and C3, alternating.
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/r1_C2.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/r1_C2.json'));print('C2 r1 run $i', d['ms_per_step'], d['solve']['a_matvecs_per_solve'], d['clocks']['sm_mhz'])")
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/r2_C2.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/r2_C2.json'));print('C2 r2 run $i', d['ms_per_step'], d['solve']['a_matvecs_per_solve'], d['clocks']['sm_mhz'])"
done
for i in 1 2; do
  (cd baseline/r1 && timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/r1_C3.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/r1_C3.json'));print('C3 r1 run $i', d['ms_per_step'], d['solve']['a_matvecs_per_solve'], d['clocks']['sm_mhz'])")
  timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/r2_C3.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/r2_C3.json'));print('C3 r2 run $i', d['ms_per_step'], d['solve']['a_matvecs_per_solve'], d['clocks']['sm_mhz'])"
done

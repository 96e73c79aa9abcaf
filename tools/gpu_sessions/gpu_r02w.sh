#!/bin/bash
# Round-1 tree vs current (C2 / C3, alternating); multi-rank parity with the halo overlap.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json,sys;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for i in 1 2 3; do
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/r1_C2.json 2>/tmp/r1_C2.err); pr /tmp/r1_C2.json "C2 r1 run $i"
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/r2_C2.json 2>/dev/null; pr /tmp/r2_C2.json "C2 r2 run $i"
done
tail -3 /tmp/r1_C2.err
for i in 1 2; do
  (cd baseline/r1 && timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/r1_C3.json 2>/dev/null); pr /tmp/r1_C3.json "C3 r1 run $i"
  timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/r2_C3.json 2>/dev/null; pr /tmp/r2_C3.json "C3 r2 run $i"
done
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_torchrun.py -q -x > $O/r02w_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02w_pytest.log

#!/bin/bash
# New tests (quasi-optimality diagnostic, pipelined rotation), rotation alone new vs HEAD~ tree, C3 solve A/B.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pl1.py tests/test_gpu_multirank.py tests/test_gpu_kernels.py -q -rf --timeout 600 -k "quasi or pl1_loopback or rotate" > $O/rot_pytest.log 2>&1; echo "pytest rc=$?" >> $O/rot_pytest.log; tail -3 $O/rot_pytest.log
for a in "C3 48 20" "C3 32 20" "C5 24 10" "C2 30 12"; do
  timeout 300 python tools/rot_time.py $a 20 2>&1 | tail -1 | sed 's/^/new /'
  (cd baseline/r2h && timeout 300 python tools/rot_time.py $a 20 2>&1 | tail -1 | sed 's/^/old /')
done
pr() { python -c "import json,sys;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline'].get('cycle_phases_ms'))" 2>&1 | tail -1; }
for i in 1 2; do
  timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C3 new $i"
  (cd baseline/r2h && timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /tmp/b.json 2>/dev/null); pr /tmp/b.json "C3 old $i"
done

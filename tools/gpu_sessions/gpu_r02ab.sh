#!/bin/bash
# +K first pass on the preceding K1 (set2 = 4), mat_row back to round-1 form: parity + C2/C3/C5 lines.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json,sys;d=json.load(open('$1'));r=d['roofline'];print('$2', d['ms_per_step'], d['clocks']['sm_mhz'], r['cycle_phases_ms'])" 2>&1 | tail -1; }
timeout 1200 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py tests/test_gpu_multirank.py tests/test_gpu_branches.py tests/test_gpu_fullsize.py -q -x -m gpu > $O/r02ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02ab_pytest.log
for i in 1 2; do
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C2 main run $i"
  (cd baseline/r1 && timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/c.json 2>/dev/null); python -c "import json;d=json.load(open('/tmp/c.json'));print('C2 r1', d['ms_per_step'])"
done
timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/a.json 2>/dev/null; pr /tmp/a.json "C3 main"
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > $O/r02ab_C5.json 2>/dev/null; pr $O/r02ab_C5.json "C5 main"

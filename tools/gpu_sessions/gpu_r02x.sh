#!/bin/bash
# C2 regression hunt: round-1 tree vs current, per-kernel launch lists of one timed C2 solve; env switches.
O=gpurun_out; mkdir -p $O
pr() { python -c "import json,sys;d=json.load(open('$1'));print('$2', d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for v in default tpdots; do
  if [ $v = default ]; then unset TRPLK_K1; else export TRPLK_K1=$v; fi
  timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-last-only > /tmp/x.json 2>/dev/null; pr /tmp/x.json "C2 r2 K1=$v"
done
unset TRPLK_K1
TRPLK_HALO_OVERLAP=1 timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -k halo_overlap > $O/r02x_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/r02x_pytest.log
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file $O/r02x_r2_C2_launches.csv python tools/solve_twice.py C2 > $O/r02x_r2_ncu.log 2>&1
python tools/launch_sum.py $O/r02x_r2_C2_launches.csv > $O/r02x_r2_C2_sum.txt 2>&1; head -25 $O/r02x_r2_C2_sum.txt
(cd baseline/r1 && ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv --log-file ../../$O/r02x_r1_C2_launches.csv python tools/solve_twice.py C2 > ../../$O/r02x_r1_ncu.log 2>&1)
python tools/launch_sum.py $O/r02x_r1_C2_launches.csv > $O/r02x_r1_C2_sum.txt 2>&1; head -25 $O/r02x_r1_C2_sum.txt

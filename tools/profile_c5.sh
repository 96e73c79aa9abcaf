#!/bin/bash
# C5 ncu evidence (run on the GPU box): launch list of a steady window of one solve, --set full of
# the three inner-step kernels, traffic_C5.json.  The plain bench must have exited 0 first.
set -u
O=gpurun_out
B="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $O/r02_plain_C5.json 2> $O/r02_plain_C5.err || { echo "plain run failed"; tail -5 $O/r02_plain_C5.err; exit 1; }
# launch list: skip start-up and the first solve (~17k launches each), then 1600 launches (~10 cycles)
ncu --metrics gpu__time_duration.sum --clock-control none -s 20000 -c 1600 --csv \
    --log-file $O/r02_launches_C5.csv $B > $O/r02_ncu_launch_C5.log 2>&1
python tools/launch_sum.py $O/r02_launches_C5.csv > $O/r02_C5_launches_summary.txt 2>&1
ncu -f --set full --clock-control none --import-source on \
    -k regex:'k_step1_pipe|k_upd2_wp2|k_upd<|k_rotate_s|k_step1_tp|k_eig' -s 2000 -c 14 \
    -o /tmp/prof_C5 $B > $O/r02_ncu_full_C5.log 2>&1
python tools/ncu_summary.py rep /tmp/prof_C5.ncu-rep > $O/r02_C5_ncu_full_summary.txt 2>&1
python tools/ncu_source_top.py /tmp/prof_C5.ncu-rep . 25 > $O/r02_C5_ncu_source_top.txt 2>&1
rm -f profiles/traffic_C5.json
python tools/make_traffic.py /tmp/prof_C5.ncu-rep C5 > $O/r02_traffic_C5.log 2>&1
cp profiles/traffic_C5.json $O/ 2>/dev/null
cp /tmp/prof_C5.ncu-rep $O/r02_prof_C5.ncu-rep 2>/dev/null
tail -n 2 $O/r02_ncu_*_C5.log

#!/bin/bash
# Run on the GPU box (gpurun): plain bench, ncu launch list, ncu --set full of the inner-step
# kernels (summarised on the box: reports are not copied back), traffic_<cfg>.json.
#   gpurun -- 'bash tools/profile_round.sh C2'
set -u
CFG=${1:-C2}
OUT=gpurun_out
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $OUT/plain_$CFG.json 2> $OUT/plain_$CFG.err || { echo "plain run failed"; tail -5 $OUT/plain_$CFG.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file $OUT/launches_$CFG.csv $B > $OUT/ncu_launch_$CFG.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:'k_(step1|upd|rotate|eig)' -s 600 -c 30 \
    -o /tmp/prof_$CFG $B > $OUT/ncu_full_$CFG.log 2>&1
python tools/ncu_summary.py rep /tmp/prof_$CFG.ncu-rep > $OUT/ncu_full_summary_$CFG.txt 2>&1
python tools/ncu_source_top.py /tmp/prof_$CFG.ncu-rep . 25 > $OUT/ncu_source_top_$CFG.txt 2>&1
python tools/make_traffic.py /tmp/prof_$CFG.ncu-rep $CFG > $OUT/traffic_$CFG.log 2>&1
cp profiles/traffic_$CFG.json $OUT/ 2>/dev/null
tail -n 2 $OUT/ncu_*_$CFG.log

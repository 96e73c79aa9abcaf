#!/bin/bash
# C5 ncu evidence (run on the GPU box): launch list of a steady window of one solve, --set full of
# the three inner-step kernels, traffic_C5.json.  The plain bench must have exited 0 first.
set -u
O=gpurun_out
B="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $O/r02_plain_C5.json 2> $O/r02_plain_C5.err || { echo "plain run failed"; tail -5 $O/r02_plain_C5.err; exit 1; }
# launch list: skip start-up and most of the first (warm-up) solve (~5,700 launches per solve), then
# 1,600 launches (~30 steady cycles of the timed solve)
ncu --metrics gpu__time_duration.sum --clock-control none -s 7000 -c 1600 --csv \
    --log-file $O/r02_launches_C5.csv $B > $O/r02_ncu_launch_C5.log 2>&1
python tools/launch_sum.py $O/r02_launches_C5.csv > $O/r02_C5_launches_summary.txt 2>&1
# --set full of the inner-step kernels K1 / K2 / K3 (3 launches each, mid-solve) and of the
# per-cycle seed / +K dot kernel and rotation (one each)
rm -f profiles/traffic_C5.json
for K in 'k_step1_pipe<16' 'k_upd2_wp2<8' 'k_upd<16' 'k_step1_tp<24' 'k_rotate_s'; do
  tag=$(echo "$K" | tr -c 'a-z0-9_' '_')
  C=3; case $K in k_step1_tp*|k_rotate_s*) C=1;; esac
  ncu -f --set full --clock-control none --import-source on -k regex:"$K" -s 300 -c $C \
      -o /tmp/prof_C5_$tag $B > $O/r02_ncu_full_C5_$tag.log 2>&1
  python tools/ncu_summary.py rep /tmp/prof_C5_$tag.ncu-rep >> $O/r02_C5_ncu_full_summary.txt 2>&1
  python tools/make_traffic.py /tmp/prof_C5_$tag.ncu-rep C5 >> $O/r02_traffic_C5.log 2>&1
done
python tools/ncu_source_top.py /tmp/prof_C5_k_step1_pipe_16.ncu-rep . 25 > $O/r02_C5_ncu_source_top.txt 2>&1
cp /tmp/prof_C5_k_step1_pipe_16.ncu-rep $O/r02_prof_C5_K1.ncu-rep 2>/dev/null
cp profiles/traffic_C5.json $O/ 2>/dev/null
tail -n 2 $O/r02_ncu_*_C5.log

#!/bin/bash
# Round-2 final measurement: C5 ncu (launch list + --set full of the inner-step kernels ->
# traffic_C5.json), then the driver-default bench line (C5, e2e, cpu_baseline), the other configs,
# the reference arm, smoke.
set -u
O=gpurun_out; mkdir -p $O
B="python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $O/fin_plain_C5.json 2> $O/fin_plain_C5.err || { echo "plain run failed"; tail -5 $O/fin_plain_C5.err; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 7000 -c 1600 --csv \
    --log-file $O/fin_launches_C5.csv $B > $O/fin_ncu_launch_C5.log 2>&1
python tools/launch_sum.py $O/fin_launches_C5.csv > $O/fin_C5_launches_summary.txt 2>&1; head -20 $O/fin_C5_launches_summary.txt
rm -f profiles/traffic_C5.json $O/fin_C5_ncu_full_summary.txt $O/fin_traffic_C5.log
for K in 'k_step1_lean<16' 'k_step1_rs2<24' 'k_upd2_wp2<8' 'k_upd<16' 'k_upd2_wp2<12' 'k_upd<24' 'k_rotate_s' 'k_step1_tp<24'; do
  tag=$(echo "$K" | tr -c 'a-z0-9_' '_')
  C=2; case $K in k_step1_tp*|k_rotate_s*) C=1;; esac
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$K" -s 40 -c $C \
      -o /tmp/fin_C5_$tag $B > $O/fin_ncu_full_C5_$tag.log 2>&1
  python tools/ncu_summary.py rep /tmp/fin_C5_$tag.ncu-rep >> $O/fin_C5_ncu_full_summary.txt 2>&1
  python tools/make_traffic.py /tmp/fin_C5_$tag.ncu-rep C5 >> $O/fin_traffic_C5.log 2>&1
done
python tools/ncu_source_top.py /tmp/fin_C5_k_step1_lean_16.ncu-rep . 25 > $O/fin_C5_K1_source_top.txt 2>&1
cp profiles/traffic_C5.json $O/fin_traffic_C5.json 2>/dev/null
cut -c1-400 $O/fin_C5_ncu_full_summary.txt
timeout 1500 python bench.py > $O/fin_bench_default.json 2> $O/fin_bench_default.err; echo "default bench rc=$?"; cat $O/fin_bench_default.json | cut -c1-600
for c in C1 C2 C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/fin_bench_$c.json 2> $O/fin_bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --config C2 > $O/fin_bench_C2_cpu.json 2> /dev/null; echo "C2 with cpu_baseline rc=$?"
timeout 1800 python bench.py --impl reference --steps 2 --warmup 1 > $O/fin_ref_C5.json 2> $O/fin_ref_C5.err; echo "reference rc=$?"; cat $O/fin_ref_C5.json | cut -c1-400
timeout 300 python __graft_entry__.py --smoke > $O/fin_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/fin_smoke.log

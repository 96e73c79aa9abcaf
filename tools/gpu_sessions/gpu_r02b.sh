#!/bin/bash
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $O/r02b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r02b_pytest_gpu.log
tail -3 $O/r02b_pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02b_bench_C5.json 2> $O/r02b_bench_C5.err; echo "bench rc=$?"
# ncu --set full of the C5 inner-step kernels launched alone (tools/c5_kernels.py)
rm -f profiles/traffic_C5.json
for K in 'k_step1_pipe' 'k_upd2_wp2' 'k_upd<' 'k_step1_tp' 'k_rotate_s'; do
  tag=$(echo "$K" | tr -c 'a-z0-9_' '_')
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 2 \
      -o /tmp/prof_C5_$tag python tools/c5_kernels.py 2 > $O/r02b_ncu_full_C5_$tag.log 2>&1
  python tools/ncu_summary.py rep /tmp/prof_C5_$tag.ncu-rep >> $O/r02b_C5_ncu_full_summary.txt 2>&1
  python tools/make_traffic.py /tmp/prof_C5_$tag.ncu-rep C5 >> $O/r02b_traffic_C5.log 2>&1
done
python tools/ncu_source_top.py /tmp/prof_C5_k_step1_pipe.ncu-rep . 25 > $O/r02b_C5_ncu_source_top.txt 2>&1
cp /tmp/prof_C5_k_step1_pipe.ncu-rep $O/r02b_prof_C5_K1.ncu-rep 2>/dev/null
cp profiles/traffic_C5.json $O/ 2>/dev/null
# how long does an ncu launch list take on a C3 solve (graphs, ~10k launches)?
S=$(date +%s)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02b_launches_C3.csv \
   python bench.py --config C3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/r02b_ncu_launch_C3.log 2>&1
echo "C3 launch list rc=$? $(( $(date +%s) - S )) s"
python tools/launch_sum.py $O/r02b_launches_C3.csv > $O/r02b_C3_launches_summary.txt 2>&1

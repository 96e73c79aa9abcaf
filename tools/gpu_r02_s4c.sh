#!/bin/bash
# Session-4 call 3: ncu --set full of the C5 kernel instantiations launched alone (tools/c5_kernels.py) ->
# traffic_C5.json; default bench line (C5) with the SURVEY 8(d) algorithmic byte model; C2 / C3 / C4 lines;
# the whole GPU suite at HEAD.
O=gpurun_out; mkdir -p $O
timeout 300 python tools/c5_kernels.py 1 > $O/s4c_c5_kernels.log 2>&1; echo "c5_kernels rc=$?"; tail -8 $O/s4c_c5_kernels.log
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:'k_step1_lean|k_step1_rs2|k_step1_pipe|k_upd|k_upd2_wp2|k_rotate_s|k_step1_tp' -c 24 \
    -o /tmp/s4c_C5 python tools/c5_kernels.py 1 > $O/s4c_ncu_full_C5.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py rep /tmp/s4c_C5.ncu-rep > $O/s4c_C5_ncu_full_summary.txt 2>&1
python tools/make_traffic.py /tmp/s4c_C5.ncu-rep C5 > $O/s4c_traffic_C5.log 2>&1
cp profiles/traffic_C5.json $O/s4c_traffic_C5.json 2>/dev/null
python tools/ncu_source_top.py /tmp/s4c_C5.ncu-rep . 25 > $O/s4c_C5_source_top.txt 2>&1
cut -c1-330 $O/s4c_C5_ncu_full_summary.txt
timeout 1500 python bench.py > $O/s4c_bench_default.json 2> $O/s4c_bench_default.err; echo "default bench rc=$?"; cut -c1-1200 $O/s4c_bench_default.json
for c in C2 C3 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline > $O/s4c_bench_$c.json 2> $O/s4c_bench_$c.err; echo "$c rc=$?"; done
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/s4c_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/s4c_pytest_gpu.log
tail -4 $O/s4c_pytest_gpu.log

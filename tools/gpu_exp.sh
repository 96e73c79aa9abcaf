mkdir -p gpurun_out/exp
O=gpurun_out/exp
B="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $O/plain.json 2> $O/plain.err || exit 1
ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_step1_rs2<.int.24, .bool.1>' -c 3 -o /tmp/k1 $B > $O/ncu_k1.log 2>&1
python tools/ncu_summary.py rep /tmp/k1.ncu-rep > $O/k1_summary.txt 2>&1
python tools/ncu_source_top.py /tmp/k1.ncu-rep . 30 > $O/k1_source_top.txt 2>&1
python tools/make_traffic.py /tmp/k1.ncu-rep C2 > $O/k1_traffic.log 2>&1
B3="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
ncu -f --set full --clock-control none --kernel-name-base demangled -k regex:'k_step1_rs2<.int.32, .bool.1>' -s 20 -c 3 -o /tmp/k3 $B3 > $O/ncu_k3.log 2>&1
python tools/make_traffic.py /tmp/k3.ncu-rep C3 > $O/k3_traffic.log 2>&1
python tools/ncu_summary.py rep /tmp/k3.ncu-rep > $O/k3_summary.txt 2>&1
cp profiles/traffic_C2.json profiles/traffic_C3.json $O/

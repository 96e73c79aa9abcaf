#!/bin/bash
# ncu --set full of every streaming kernel at C3 (k = 45) and C2 (k = 24) sizes, launched alone
O=gpurun_out
for CK in "C3 45" "C2 24"; do
  set -- $CK; C=$1; K=$2
  timeout 900 ncu -f --set full --clock-control none --import-source on \
     -k regex:'k_step1|k_upd|k_rotate|k_blk' -s 12 -c 12 -o /tmp/kern_$C python tools/kernels_at.py $C $K 2 > $O/r02g_ncu_$C.log 2>&1
  python tools/ncu_summary.py rep /tmp/kern_$C.ncu-rep > $O/r02g_${C}_kernels_ncu_summary.txt 2>&1
done
for C in C2 C3; do
  TRPLK_KPLUS=col timeout 900 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/r02g_bench_${C}_col.json 2> $O/r02g_bench_${C}_col.err
  timeout 900 python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $O/r02g_bench_${C}_blk.json 2> $O/r02g_bench_${C}_blk.err
done
echo done-all

#!/bin/bash
O=gpurun_out
python tools/blk_micro.py 24 2 3 > $O/r02e_blk_micro.txt 2>&1
python tools/blk_micro.py 16 2 3 >> $O/r02e_blk_micro.txt 2>&1
cat $O/r02e_blk_micro.txt
for M in 'k_blk<24, 0>' 'k_blk<24, 1>' 'k_blk<24, 2>'; do
  tag=$(echo "$M" | tr -c 'a-z0-9_' '_')
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"k_blk" --kernel-name-base demangled -c 3 -o /tmp/blk_$tag python tools/blk_micro.py 24 2 1 > $O/r02e_ncu_$tag.log 2>&1
  python tools/ncu_summary.py rep /tmp/blk_$tag.ncu-rep >> $O/r02e_blk_ncu_summary.txt 2>&1
  break
done
python tools/ncu_source_top.py /tmp/blk_k_blk_24__0_.ncu-rep . 30 > $O/r02e_blk_source_top.txt 2>&1
for B in 2 3; do
  timeout 900 python bench.py --config C5 --block $B --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02e_bench_C5_b$B.json 2> $O/r02e_bench_C5_b$B.err; echo "bench C5 b$B rc=$?"
done

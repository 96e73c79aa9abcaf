#!/bin/bash
O=gpurun_out
echo "== LB1" > $O/r02f_blk_micro.txt
python tools/blk_micro.py 24 2 3 >> $O/r02f_blk_micro.txt 2>&1
python tools/blk_micro.py 16 2 3 >> $O/r02f_blk_micro.txt 2>&1
echo "== LB2" >> $O/r02f_blk_micro.txt
TRPLK_BLK_LB=2 python tools/blk_micro.py 24 2 3 >> $O/r02f_blk_micro.txt 2>&1
TRPLK_BLK_LB=2 python tools/blk_micro.py 16 2 3 >> $O/r02f_blk_micro.txt 2>&1
echo "== KPLUS=col C5 bench" >> $O/r02f_blk_micro.txt
cat $O/r02f_blk_micro.txt
timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02f_bench_C5_lb1.json 2> $O/r02f_bench_C5_lb1.err; echo "lb1 rc=$?"
TRPLK_BLK_LB=2 timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02f_bench_C5_lb2.json 2> $O/r02f_bench_C5_lb2.err; echo "lb2 rc=$?"
TRPLK_KPLUS=col timeout 900 python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02f_bench_C5_col.json 2> $O/r02f_bench_C5_col.err; echo "col rc=$?"

#!/bin/bash
# Fused K3+K1 v2 (interleaved loads, grid semaphore): parity subset, A/B vs the 3-kernel step, ncu of the fused kernel.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_branches.py -q -x -m gpu > $O/r02q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02q_pytest.log
timeout 300 python tools/ab.py C2 "TRPLK_FUSE=0" "" 5 > $O/r02q_ab_C2_fuse.txt 2>&1; tail -3 $O/r02q_ab_C2_fuse.txt
timeout 400 python tools/ab.py C3 "TRPLK_FUSE=0" "" 3 > $O/r02q_ab_C3_fuse.txt 2>&1; tail -3 $O/r02q_ab_C3_fuse.txt
B="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:'k_fin_step1|k_upd2_wp2|k_step1_rs2' -s 300 -c 6 -o /tmp/fz_C3 $B > $O/r02q_ncu_C3.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py rep /tmp/fz_C3.ncu-rep > $O/r02q_ncu_C3_summary.txt 2>&1; cat $O/r02q_ncu_C3_summary.txt | cut -c1-600
python tools/ncu_source_top.py /tmp/fz_C3.ncu-rep . 30 > $O/r02q_ncu_C3_source.txt 2>&1
cp /tmp/fz_C3.ncu-rep $O/r02q_fz_C3.ncu-rep
timeout 900 python tools/ab.py C5 "TRPLK_FUSE=0" "" 1 > $O/r02q_ab_C5_fuse.txt 2>&1; tail -3 $O/r02q_ab_C5_fuse.txt

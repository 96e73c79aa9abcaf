#!/bin/bash
# Run on the GPU box (gpurun): plain bench, ncu launch list, ncu --set full of the inner-step
# kernels.  Outputs in gpurun_out/; summarise here with tools/ncu_summary.py into profiles/.
#   gpurun -- 'bash tools/profile_round.sh C2'
set -u
CFG=${1:-C2}
OUT=gpurun_out
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $OUT/plain_$CFG.json 2> $OUT/plain_$CFG.err || { echo "plain run failed"; tail -5 $OUT/plain_$CFG.err; exit 1; }
# launch list of one cycle's worth of kernels after warm-up (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file $OUT/launches_$CFG.csv $B > $OUT/ncu_launch_$CFG.log 2>&1
# top kernels, one launch each (K1 = k_sdots_mma with two dot sets, K2/K3 = k_upd)
ncu --set full --clock-control none --import-source on -k regex:k_sdots_mma -s 300 -c 1 \
    -o $OUT/prof_K1_$CFG $B > $OUT/ncu_K1_$CFG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_upd -s 300 -c 3 \
    -o $OUT/prof_K23_$CFG $B > $OUT/ncu_K23_$CFG.log 2>&1
tail -n 2 $OUT/ncu_*_$CFG.log

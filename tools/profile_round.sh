#!/bin/bash
# Run on the GPU box (gpurun): plain bench, ncu launch list, ncu --set full of the inner-step
# kernels and the Rayleigh-Ritz eig.  Outputs in gpurun_out/; summarise here with
# tools/ncu_summary.py into profiles/.
#   gpurun -- 'bash tools/profile_round.sh C2'
set -u
CFG=${1:-C2}
OUT=gpurun_out
B="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > $OUT/plain_$CFG.json 2> $OUT/plain_$CFG.err || { echo "plain run failed"; tail -5 $OUT/plain_$CFG.err; exit 1; }
# launch list of the second solve's first cycles (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
    --log-file $OUT/launches_$CFG.csv $B > $OUT/ncu_launch_$CFG.log 2>&1
# top kernels: K1 (fused SpMV + Jacobi + dots), K2 (CGS pass 2), K3 (final update), eig
ncu --set full --clock-control none --import-source on -k regex:'^k_(step1_tp|upd2_tp|upd|eig)$' -s 600 -c 8 \
    -o $OUT/prof_$CFG $B > $OUT/ncu_full_$CFG.log 2>&1
tail -n 2 $OUT/ncu_*_$CFG.log

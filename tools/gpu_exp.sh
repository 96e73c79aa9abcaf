mkdir -p gpurun_out/exp
O=gpurun_out/exp
TRPLK_TIMING=1 python tools/solve_twice.py C2 > $O/timing.txt 2>&1

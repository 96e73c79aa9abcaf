mkdir -p gpurun_out/exp
O=gpurun_out/exp
TRPLK_CYCLE_TRACE=1 python tools/solve_twice.py C2 > $O/ctrace.txt 2>&1
TRPLK_CYCLE_TRACE=1 python tools/solve_twice.py C3 >> $O/ctrace.txt 2>&1

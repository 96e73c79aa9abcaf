mkdir -p gpurun_out/exp
O=gpurun_out/exp
TRPLK_EIG=tri TRPLK_EIG_NEV=10 python tools/eig_time.py > $O/eig_tri_clk.txt 2>&1
TRPLK_EIG=tri python tools/eig_time.py > $O/eig_tri_full.txt 2>&1

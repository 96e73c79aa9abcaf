mkdir -p gpurun_out/exp
O=gpurun_out/exp
python tools/k1_scaling.py > $O/k1_scaling.txt 2>&1

mkdir -p gpurun_out/exp
O=gpurun_out/exp
for E in TRPLK_NO_COOP3=1 TRPLK_NO_SMALL=1 TRPLK_GRID=1 TRPLK_KVAR=tp TRPLK_K2=rs; do
  echo "== $E" >> $O/alt.log
  env $E timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_multirank.py -m gpu -q -x --timeout 300 2>&1 | tail -2 >> $O/alt.log
done

#!/bin/bash
# K1 variants alone after DIA-C constants moved into the descriptor (kernel parameters).
O=gpurun_out; mkdir -p $O
for cfg in "C5 15" "C5 23" "C3 15" "C3 23" "C3 31"; do
  for v in pipe rs lean; do
    for dc in 1 0; do
      TRPLK_DIAC=$dc TRPLK_K1=$v timeout 300 python tools/k1_time.py $cfg 10 2>&1 | tail -1
    done
  done
done > $O/r02t_k1_time.txt; cat $O/r02t_k1_time.txt
timeout 600 python -m pytest tests/test_gpu_solve.py -q -x -k "dia_constant" > $O/r02t_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/r02t_pytest.log

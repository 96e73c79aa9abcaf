#!/bin/bash
# Lean K1 + DIA-C default at C5 k <= 16: full GPU suite, interleaved A/B at C5 (DIAC off = pipe).
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/r02ac_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/r02ac_pytest.log
timeout 1200 python tools/ab.py C5 "TRPLK_DIAC=0" "" 2 > $O/r02ac_ab_C5.txt 2>&1; tail -3 $O/r02ac_ab_C5.txt

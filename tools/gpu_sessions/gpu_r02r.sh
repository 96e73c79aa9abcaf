#!/bin/bash
# DIA-C A/B on the default (unfused) path; full GPU suite.
O=gpurun_out; mkdir -p $O
timeout 300 python tools/ab.py C2 "TRPLK_DIAC=0" "" 5 > $O/r02r_ab_C2_diac.txt 2>&1; tail -3 $O/r02r_ab_C2_diac.txt
timeout 400 python tools/ab.py C3 "TRPLK_DIAC=0" "" 3 > $O/r02r_ab_C3_diac.txt 2>&1; tail -3 $O/r02r_ab_C3_diac.txt
timeout 900 python tools/ab.py C5 "TRPLK_DIAC=0" "" 2 > $O/r02r_ab_C5_diac.txt 2>&1; tail -3 $O/r02r_ab_C5_diac.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/r02r_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r02r_pytest.log

#!/bin/bash
# Fused K3+K1 (k_fin_step1) parity: full GPU suite; interleaved A/B of FUSE and DIAC at C3 / C5.
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf --timeout 900 > $O/r02p_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/r02p_pytest.log
timeout 300 python tools/ab.py C2 "TRPLK_FUSE=0" "" 5 > $O/r02p_ab_C2_fuse.txt 2>&1; cat $O/r02p_ab_C2_fuse.txt | tail -3
timeout 400 python tools/ab.py C3 "TRPLK_FUSE=0" "" 3 > $O/r02p_ab_C3_fuse.txt 2>&1; cat $O/r02p_ab_C3_fuse.txt | tail -3
timeout 400 python tools/ab.py C3 "TRPLK_DIAC=0" "" 3 > $O/r02p_ab_C3_diac.txt 2>&1; cat $O/r02p_ab_C3_diac.txt | tail -3
timeout 600 python tools/ab.py C4 "TRPLK_DIAC=0" "" 2 > $O/r02p_ab_C4_diac.txt 2>&1; cat $O/r02p_ab_C4_diac.txt | tail -3
timeout 900 python tools/ab.py C5 "TRPLK_FUSE=0" "" 2 > $O/r02p_ab_C5_fuse.txt 2>&1; cat $O/r02p_ab_C5_fuse.txt | tail -3
timeout 900 python tools/ab.py C5 "TRPLK_DIAC=0" "" 2 > $O/r02p_ab_C5_diac.txt 2>&1; cat $O/r02p_ab_C5_diac.txt | tail -3

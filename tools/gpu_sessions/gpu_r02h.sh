#!/bin/bash
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r02h_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r02h_pytest_gpu.log
tail -15 $O/r02h_pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/r02h_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/r02h_smoke.log

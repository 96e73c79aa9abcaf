mkdir -p gpurun_out/exp
O=gpurun_out/exp
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 600 > $O/pytest_all.log 2>&1; echo "pytest rc=$?" >> $O/pytest_all.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err

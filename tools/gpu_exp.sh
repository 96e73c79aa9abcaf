mkdir -p gpurun_out/exp
O=gpurun_out/exp
TRPLK_KVAR=cp timeout 1500 python -m pytest tests -m gpu -q -x -rf --timeout 900 > $O/pytest_cp.log 2>&1; echo "pytest rc=$?" >> $O/pytest_cp.log
Q="--steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
for cfg in C2 C3; do
  TRPLK_KVAR=cp timeout 600 python bench.py --config $cfg $Q > $O/b_${cfg}_cp.json 2>&1
  timeout 600 python bench.py --config $cfg $Q > $O/b_${cfg}_rs.json 2>&1
done

mkdir -p gpurun_out/exp
O=gpurun_out/exp
rm -f $O/sweep.txt
for E in X=0 TRPLK_EIG_EPS=1e-14 TRPLK_EIG_EPS=1e-12; do for C in C2 C3; do
echo "== $E $C" >> $O/sweep.txt
env $E python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>>$O/sweep.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['config']['a_matvecs_per_solve'], d['config']['cycles'])" >> $O/sweep.txt
done; done
TRPLK_EIG_EPS=1e-14 timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -q --timeout 600 > $O/pytest_eps.log 2>&1; echo "rc=$?" >> $O/pytest_eps.log

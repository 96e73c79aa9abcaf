mkdir -p gpurun_out/exp
O=gpurun_out/exp
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
for c in C2 C3; do timeout 600 python bench.py --method pl1 --config $c > $O/bench_pl1_$c.json 2> $O/bench_pl1_$c.err; done

# round-2 refresh: full GPU suite (parity metrics), smoke, bench lines c1..c5 + reference arms, c2 launch list
FL1_PARITY_OUT=gpurun_out/parity_final.json timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/final_tests.log 2>&1
echo tests_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke_rc=$?
for c in c1 c2 c3 c5 c4; do
  timeout 900 python bench.py --config $c > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err; echo bench_${c}_rc=$?
done
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --impl reference --config $c > gpurun_out/final_ref_$c.json 2> gpurun_out/final_ref_$c.err; echo ref_${c}_rc=$?
done
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_c4.log 2>&1; echo ncu_rc=$?

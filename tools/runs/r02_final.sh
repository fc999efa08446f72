# round-2 final refresh: GPU suite (parity records), smoke, bench lines c1..c5 (c4 as the driver runs it),
# reference arms, launch list of the default bench line
FL1_PARITY_OUT=gpurun_out/parity_final3.json timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final3_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/final3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo smoke_rc=$?; cat gpurun_out/final3_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final3_bench_c4.json 2> gpurun_out/final3_bench_c4.err; echo bench_c4_rc=$?
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/final3_bench_$c.json 2> gpurun_out/final3_bench_$c.err; echo bench_${c}_rc=$?
done
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final3_ref_c4.json 2> gpurun_out/final3_ref_c4.err; echo ref_c4_rc=$?
for c in c1 c2 c3 c5; do
  timeout 900 python bench.py --impl reference --config $c --steps 5 --warmup 1 > gpurun_out/final3_ref_$c.json 2> gpurun_out/final3_ref_$c.err; echo ref_${c}_rc=$?
done
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final3_launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final3_ncu_c4.log 2>&1; echo ncu_rc=$?

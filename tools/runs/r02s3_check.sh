# session-3 re-entry check: rebuilt tree on a fresh box (GPU suite, smoke, c2 / c5 short bench lines)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/s3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
for c in c2 c5 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3_bench_$c.json 2> gpurun_out/s3_bench_$c.err; echo bench_${c}_rc=$?
done

# session-3 refresh: GPU suite (parity records), smoke, bench lines c4 (as the driver runs it) and c1-c3, c5,
# c5 lockstep ncu capture and launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
FL1_PARITY_OUT=gpurun_out/s3f_parity.json timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s3f_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/s3f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3f_smoke.log 2>&1; echo smoke_rc=$?; cat gpurun_out/s3f_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3f_bench_c4.json 2> gpurun_out/s3f_bench_c4.err; echo bench_c4_rc=$?
for c in c5 c1 c2 c3; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/s3f_bench_$c.json 2> gpurun_out/s3f_bench_$c.err; echo bench_${c}_rc=$?
done
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:prefix_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/s3f_c5_prefix python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3f_ncu_c5.log 2>&1; echo ncu_c5_rc=$?
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3f_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3f_ncu_c5_launches.log 2>&1; echo ncu_launches_rc=$?

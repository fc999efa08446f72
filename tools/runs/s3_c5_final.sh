# c5 after the shared-memory operand fix: GPU suite subset, bench line, step log, ncu capture, launch list
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s3g_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/s3g_tests.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 5 > gpurun_out/s3g_bench_c5.json 2> gpurun_out/s3g_bench_c5.err; echo bench_rc=$?
timeout 180 python tools/step_log.py > gpurun_out/s3g_c5_steplog.txt 2>&1; tail -14 gpurun_out/s3g_c5_steplog.txt
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:prefix_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/s3g_c5_prefix python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3g_ncu_c5.log 2>&1; echo ncu_rc=$?
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3g_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3g_ncu_c5_launches.log 2>&1; echo ncu_launches_rc=$?

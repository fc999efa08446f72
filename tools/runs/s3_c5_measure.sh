# c5 with the stream-K lockstep: GPU suite, bench line, step log, ncu capture of the lockstep launch
FL1_PARITY_OUT=gpurun_out/s3_parity.json timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s3_suite.log 2>&1; echo suite_rc=$?; tail -3 gpurun_out/s3_suite.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 5 > gpurun_out/s3_bench_c5.json 2> gpurun_out/s3_bench_c5.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/s3_bench_c5.json').read()); print('c5', round(d['ms_per_step'],3), d['roofline']['frac'], d['roofline']['launch_ms'], d['e2e']['value'], d['clocks'])"
timeout 180 python tools/step_log.py > gpurun_out/s3_c5_steplog.txt 2>&1; tail -8 gpurun_out/s3_c5_steplog.txt
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:prefix_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/s3_c5_prefix python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s3_ncu_c5.log 2>&1; echo ncu_rc=$?

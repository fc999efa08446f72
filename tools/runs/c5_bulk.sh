timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "tile_staging" > gpurun_out/c5b_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/c5b_tests.log
FL1_LOCKSTEP_BULK=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "batched" > gpurun_out/c5b_tests2.log 2>&1; echo tests2_rc=$?; tail -3 gpurun_out/c5b_tests2.log
for v in 1 0 1 0; do
  FL1_LOCKSTEP_BULK=$v timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5b.json 2>> gpurun_out/c5b.err
  python -c "import json; d=json.loads(open('gpurun_out/c5b.json').read()); print('c5 bulk=$v', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2), d['roofline']['frac'])"
done
FL1_LOCKSTEP_BULK=1 FL1_STEP_LOG=1 timeout 300 python tools/step_log.py > gpurun_out/c5b_steplog.txt 2>&1; cat gpurun_out/c5b_steplog.txt

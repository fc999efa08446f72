timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5" > gpurun_out/pair_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/pair_tests.log
for r in 1 2; do for v in 0 1; do
  FL1_PAIR_POWER=$v timeout 300 python bench.py --config c5 --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/pair.json 2>> gpurun_out/pair.err
  python -c "import json; d=json.loads(open('gpurun_out/pair.json').read()); print('pair_power=$v', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done; done
timeout 180 python tools/step_log.py > gpurun_out/pair_steplog.txt 2>&1; tail -7 gpurun_out/pair_steplog.txt

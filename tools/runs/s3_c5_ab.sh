# c5 quick: lockstep parity subset, step log, bench
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5" > gpurun_out/ab_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/ab_tests.log
timeout 180 python tools/step_log.py > gpurun_out/ab_steplog.txt 2>&1; tail -8 gpurun_out/ab_steplog.txt
for i in 1 2; do
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c5.json 2>> gpurun_out/ab.err
python -c "import json; d=json.loads(open('gpurun_out/ab_c5.json').read()); print('c5', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2), d['clocks']['sm_mhz'])"
done

# stream-K TMA lockstep contractions: first check (hang-guarded), parity, step log A/B, bench A/B
timeout 180 python tools/step_log.py > gpurun_out/tma1_steplog.txt 2>&1; echo steplog_rc=$?; cat gpurun_out/tma1_steplog.txt | tail -12
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5" > gpurun_out/tma1_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/tma1_tests.log
FL1_LOCKSTEP_TMA=0 timeout 180 python tools/step_log.py > gpurun_out/tma0_steplog.txt 2>&1; echo steplog0_rc=$?; tail -9 gpurun_out/tma0_steplog.txt
for m in 1 0 1 0; do
FL1_LOCKSTEP_TMA=$m timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tma_c5_$m.json 2>> gpurun_out/tma.err
python -c "import json; d=json.loads(open('gpurun_out/tma_c5_$m.json').read()); print('c5 tma=$m', round(d['ms_per_step'],3), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done

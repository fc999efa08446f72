# hand-off policy A/B on c5 with the stream-K lockstep
for v in "2 0" "3 128" "3 256" "3 512" "3 1024" "2 0" "3 256"; do
  set -- $v
  FL1_LOCKSTEP_POLICY=$1 FL1_HANDOFF_S=$2 timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pol.json 2>> gpurun_out/pol.err
  python -c "import json; d=json.loads(open('gpurun_out/pol.json').read()); print('policy $1 S<=$2', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done
FL1_LOCKSTEP_POLICY=3 timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched or lockstep or config5" > gpurun_out/pol_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/pol_tests.log

timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched" > gpurun_out/c5w_tests.log 2>&1; echo tests_rc=$?
for v in "1 1" "0 1" "1 1" "0 1"; do
  set -- $v
  FL1_LOCKSTEP_WIDTH=$1 FL1_LOCKSTEP_NARROW=$2 timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --concurrency -1 > gpurun_out/c5w.json 2>> gpurun_out/c5w.err
  python -c "import json; d=json.loads(open('gpurun_out/c5w.json').read()); print('c5 width=$1 narrow=$2', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done
FL1_STEP_LOG=1 timeout 300 python tools/step_log.py > gpurun_out/c5w_steplog.txt 2>&1; cat gpurun_out/c5w_steplog.txt

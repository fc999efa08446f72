timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "batched" > gpurun_out/c5_tests.log 2>&1
echo tests_rc=$?
for m in 1 0 1 0; do
FL1_LOCKSTEP_NARROW=$m timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5_narrow_$m.json 2>> gpurun_out/c5.err
python -c "import json; d=json.loads(open('gpurun_out/c5_narrow_$m.json').read()); print('c5 narrow=$m', round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
FL1_STEP_LOG=1 timeout 300 python tools/step_log.py > gpurun_out/c5_steplog.txt 2>&1; cat gpurun_out/c5_steplog.txt
for v in r01 cur r01 cur; do
  if [ $v = r01 ]; then L=FL1_LIB=paper_1812_06635_b200/_build/libfl1cuda_r01.so; else L=; fi
  env $L timeout 300 python tools/ab_lib.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_r01_$v.json 2>>gpurun_out/c5.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_r01_$v.json').read()); print('c2 $v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done

timeout 900 python -m pytest tests/test_switches_gpu.py -q -x -k "COLSPLIT" > gpurun_out/cs_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/cs_tests.log
for t in 0 1 4000000 16000000; do
  FL1_COLSPLIT=$t timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/cs_c4.json 2> gpurun_out/cs_c4.err
  python -c "import json; d=json.loads(open('gpurun_out/cs_c4.json').read()); print('c4 colsplit=$t', round(d['ms_per_step'],2), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
done
for t in 0 1 4000000 0 1; do
  FL1_COLSPLIT=$t timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cs_c2.json 2> gpurun_out/cs_c2.err
  python -c "import json; d=json.loads(open('gpurun_out/cs_c2.json').read()); print('c2 colsplit=$t', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done

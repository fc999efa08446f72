timeout 900 python -m pytest tests/test_switches_gpu.py -q -x -k "COLSPLIT" > gpurun_out/cs2d_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/cs2d_tests.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "large_path_all" > gpurun_out/cs2d_tests2.log 2>&1; echo tests2_rc=$?; tail -1 gpurun_out/cs2d_tests2.log
for i in 1 2; do
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cs2d_c4.json 2> gpurun_out/cs2d_c4.err
python -c "import json; d=json.loads(open('gpurun_out/cs2d_c4.json').read()); print('c4', round(d['ms_per_step'],2), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
done
FL1_COLSPLIT=1 timeout 600 python tools/timeline_c4.py 2>&1 | tail -3

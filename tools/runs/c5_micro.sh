timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "batched_lockstep_prefix or lockstep_edge or full_size_config5" > gpurun_out/c5m_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/c5m_tests.log
for v in old new old new; do
  FL1_LIB=paper_1812_06635_b200/_build/libfl1cuda_$v.so timeout 600 python tools/ab_lib.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5m.json 2>> gpurun_out/c5m.err
  python -c "import json; d=json.loads(open('gpurun_out/c5m.json').read()); print('c5 $v', round(d['ms_per_step'],3), 'lockstep ms', round(d['roofline']['launch_ms'],2))"
done

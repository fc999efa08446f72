timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "dense_configs or ragged or option_matrix or large_path_all" > gpurun_out/la_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/la_tests.log
for v in r01 cur r01 cur; do
  if [ $v = r01 ]; then L=FL1_LIB=paper_1812_06635_b200/_build/libfl1cuda_r01.so; else L=; fi
  env $L timeout 300 python tools/ab_lib.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/la_c2.json 2>>gpurun_out/la.err
  python -c "import json; d=json.loads(open('gpurun_out/la_c2.json').read()); print('c2 $v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()})"
done
for v in 1 2; do
timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/la_c4.json 2> gpurun_out/la_c4.err
python -c "import json; d=json.loads(open('gpurun_out/la_c4.json').read()); print('c4', round(d['ms_per_step'],2), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
done

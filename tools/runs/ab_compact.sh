# A/B: index-gathered streaming (default) vs physically compacted preserved columns (FL1_COMPACT=1)
timeout 900 python -m pytest tests/test_switches_gpu.py -q -x > gpurun_out/ab_compact_tests.log 2>&1
echo tests_rc=$?
for cfg in c2 c3 c4; do
  for mode in 0 1 0 1; do
    FL1_COMPACT=$mode timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_compact_${cfg}_${mode}.json 2>>gpurun_out/ab_compact.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab_compact_${cfg}_${mode}.json').read()); print('$cfg', 'compact=$mode', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done

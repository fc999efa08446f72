# same-box A/B: the round-1 library vs the current build (bench c2 / c3)
for cfg in c2 c3; do
for v in r01 cur r01 cur; do
  if [ $v = r01 ]; then L=FL1_LIB=paper_1812_06635_b200/_build/libfl1cuda_r01.so; else L=; fi
  env $L timeout 300 python tools/ab_lib.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_r01_$v.json 2>>gpurun_out/ab_r01.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_r01_$v.json').read()); print('$cfg $v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['phase_ms'])"
done
done

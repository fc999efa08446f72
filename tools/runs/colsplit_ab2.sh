for t in 0 4194304 2097152 8388608 0 4194304; do
  FL1_COLSPLIT=$t timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cs_c4.json 2> gpurun_out/cs_c4.err
  python -c "import json; d=json.loads(open('gpurun_out/cs_c4.json').read()); print('c4 colsplit=$t', round(d['ms_per_step'],2), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cs_c2.json 2> gpurun_out/cs_c2.err
python -c "import json; d=json.loads(open('gpurun_out/cs_c2.json').read()); print('c2 default', round(d['ms_per_step'],3))"

for v in 2 0 3 2 0; do
  FL1_BULK_STAGES=$v timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c4b.json 2> gpurun_out/c4b.err
  python -c "import json; d=json.loads(open('gpurun_out/c4b.json').read()); print('c4 bulk_stages=$v', round(d['ms_per_step'],2), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
done

for v in 1 0 1 0; do
FL1_LIST_APPLY=$v timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/c4_la.json 2> gpurun_out/c4_la.err
python -c "import json; d=json.loads(open('gpurun_out/c4_la.json').read()); print('list_apply=$v', round(d['ms_per_step'],2), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['clocks']['sm_mhz'])"
done

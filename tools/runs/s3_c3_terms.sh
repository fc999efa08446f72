for r in 1 2; do for v in 1 2; do
  FL1_SUKRO_TERMS=$v timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t3.json 2>> gpurun_out/t3.err
  python -c "import json; d=json.loads(open('gpurun_out/t3.json').read()); print('terms=$v', round(d['ms_per_step'],3), d.get('phase_ms'))"
done; done

timeout 900 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/c4_phases.json 2> gpurun_out/c4_phases.err
python -c "import json; d=json.loads(open('gpurun_out/c4_phases.json').read()); print(d['ms_per_step'], d['phase_ms'], d['power_bytes']/1e9, d['roofline']['hot_pass'], d['clocks'])"

timeout 300 python tools/c5_probe.py > gpurun_out/c5_probe.txt 2>&1; cat gpurun_out/c5_probe.txt
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err
python -c "import json; d=json.loads(open('gpurun_out/c5_bench.json').read()); print(d['ms_per_step'], json.dumps(d['roofline']))"

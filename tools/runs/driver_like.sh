# the driver's round-end commands (default config c4): native arm, then the reference arm
start=$(date +%s)
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_native.json 2> gpurun_out/drv_native.err; echo native_rc=$? $(( $(date +%s) - start ))s
start=$(date +%s)
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.err; echo ref_rc=$? $(( $(date +%s) - start ))s
python -c "
import json
a=json.loads(open('gpurun_out/drv_native.json').read().strip().splitlines()[-1]); b=json.loads(open('gpurun_out/drv_ref.json').read().strip().splitlines()[-1])
print('native', a['value'], a['e2e']['value'], a['roofline']['frac'], a['clocks'])
print('ref', b['value'], b['steps'], b.get('per_lambda_s'), b.get('warmup_path_s'))
print('ratio', b['value']/a['value'], 'e2e ratio', b['value']/a['e2e']['value'])"

python tools/step_log.py > gpurun_out/t_c5steps.log 2>&1
for v in 1 1; do echo -n "c5 "; python bench.py --config c5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value']*1e3, d['e2e']['value']*1e3)"; done > gpurun_out/t_c5.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "batched or golden" > gpurun_out/t_tests.log 2>&1; tail -2 gpurun_out/t_tests.log
